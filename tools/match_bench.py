"""f3 throughput: match_candidates' fused tcgen05 kernel on synthetic
candidates (every interior centre of one size, so the count is fixed).

usage: python tools/match_bench.py [M] [COUNT] [ANGLE_STEP]
Prints the fused kernel's CUDA-event time per angle group and its integer
tensor-core rate (4 products of M^2 x 48 columns per candidate).
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").environ.get("SS_PKG_ROOT") or __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1707_05647_b200 import _native  # noqa: E402
from paper_1707_05647_b200.second_stage import _GROUP, _rotation_cos_sin  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 64
count = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
step = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0
L = _native.lib()
dev = torch.device("cuda:0")
W = H = 2048
rng = np.random.default_rng(1)
img = rng.integers(0, 256, (H, W), dtype=np.uint8)
tpl = rng.integers(0, 256, (m, m), dtype=np.uint8)
lo, hi = (m - 1) // 2, m // 2
xs = rng.integers(lo, W - hi, count)
ys = rng.integers(lo, H - hi, count)
rows = torch.from_numpy(np.stack([xs, ys, np.full(count, m)], 1).astype(np.int32)).to(dev)
angles = [i * step for i in range(int(round(360 / step)))]
na = len(angles)
cs, sn = _rotation_cos_sin(angles)
cs_d, sn_d = torch.from_numpy(cs).to(dev), torch.from_numpy(sn).to(dev)
pitch = int(L.ss_match_plane_pitch(W))
planes = torch.empty(3 * H * pitch, dtype=torch.uint8, device=dev)
img_d = torch.from_numpy(img).to(dev)
tpl_d = torch.from_numpy(tpl).to(dev)
s = torch.cuda.current_stream().cuda_stream
_native.check(L.ss_match_planes(img_d.data_ptr(), W, H, planes.data_ptr(), pitch, s))
bf = torch.empty(int(L.ss_match_probe_bytes(m, na)), dtype=torch.uint8, device=dev)
stats = torch.empty((na, 3), dtype=torch.int64, device=dev)
base = torch.empty(m * m, dtype=torch.uint8, device=dev)
_native.check(L.ss_match_probes(tpl_d.data_ptr(), m, m, na, cs_d.data_ptr(), sn_d.data_ptr(), bf.data_ptr(),
                                stats.data_ptr(), base.data_ptr(), s))
parts = int(L.ss_match_parts(count))
ps = torch.empty((parts, _GROUP), dtype=torch.float64, device=dev)
pi = torch.empty((parts, _GROUP), dtype=torch.int64, device=dev)
bs = torch.empty(na, dtype=torch.float64, device=dev)
bi = torch.empty(na, dtype=torch.int64, device=dev)
groups = (na + _GROUP - 1) // _GROUP


def run():
    for g in range(groups):
        _native.check(L.ss_match_fused(planes.data_ptr(), W, H, pitch, rows.data_ptr(), 3, 0, count, m, bf.data_ptr(),
                                       na, g, stats.data_ptr(), ps.data_ptr(), pi.data_ptr(), bs.data_ptr(),
                                       bi.data_ptr(), s))


run()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
kr = (m + 63) // 64 * 64
ops = 2.0 * count * m * kr * 48 * 4 * groups  # issued MACs x 2 (padded K, 48 columns, 4 products)
print(f"m={m} candidates={count} angles={na} groups={groups}: {ms:.3f} ms per match, "
      f"{ops / ms / 1e9:.1f} TOPS issued (int8), {count * na / ms / 1e3:.1f} M hypotheses/s")
