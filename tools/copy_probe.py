"""Host<->device copy rates on this box (pinned / pageable, sizes of the
e2e results): what the native session's upload and readback can reach."""
import time

import numpy as np
import torch


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / n * 1e3


dev = torch.device("cuda:0")
for mb in (1, 4, 7, 16, 64):
    n = mb << 20
    host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    page = np.random.randint(0, 255, n, dtype=np.uint8)
    pt = torch.from_numpy(page)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h2d = t(lambda: d.copy_(host, non_blocking=True))
    d2h = t(lambda: host.copy_(d, non_blocking=True))
    h2d_page = t(lambda: d.copy_(pt))
    d2h_page = t(lambda: pt.copy_(d))
    memc = t(lambda: host.copy_(pt))
    print(f"{mb:3d} MB: pinned H2D {h2d:.3f} ms ({n / h2d / 1e6:.1f} GB/s)  D2H {d2h:.3f} ms ({n / d2h / 1e6:.1f} GB/s)  "
          f"pageable H2D {h2d_page:.3f} ({n / h2d_page / 1e6:.1f})  D2H {d2h_page:.3f} ({n / d2h_page / 1e6:.1f})  "
          f"host copy (torch) {memc:.3f} ms ({n / memc / 1e6:.1f} GB/s)")
