"""A/B of the K1/K2 table build: per-plane checksums + CUDA-event timing.

Run twice (e.g. SS_BUILD_PASS1=rec and default) and compare the printed
checksums; every plane the build writes (32-bit, hi16, int64, coarse) is
hashed.  Usage: python tools/build_ab.py [--reps N] [--cases big,small,odd]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_05647_b200 import _native  # noqa: E402


def plane_hash(t: torch.Tensor, n_planes: int) -> list:
    out = []
    flat = t.view(n_planes, -1)
    for p in range(n_planes):
        x = flat[p].to(torch.int64)
        w = (torch.arange(x.numel(), device=x.device, dtype=torch.int64) & 1023) + 1
        out.append(int((x * w).sum().item()))
        del x, w
    return out


def run_case(L, W, H, mode, reps, seed):
    dev = torch.device("cuda:0")
    g = torch.Generator(device="cpu").manual_seed(seed)
    img = torch.randint(0, 256, (H, W), generator=g, dtype=torch.uint8).to(dev)
    pitch = int(L.ss_plane_pitch(W))
    p32 = torch.empty(int(L.ss_tables32_bytes(W, H)) // 4, dtype=torch.int32, device=dev)
    p64 = hi16 = coarse = None
    shifts = []
    if mode == "int64":
        p64 = torch.empty(int(L.ss_tables_bytes(W, H)) // 8, dtype=torch.int64, device=dev)
    if mode == "hi16":
        hi16 = torch.empty(int(L.ss_tables_hi16_bytes(W, H)) // 2, dtype=torch.int16, device=dev)
    if mode in ("hi16", "u32c"):
        shifts = [4, 7, 10, 13]
        coarse = torch.empty(int(L.ss_coarse_bytes(W, H, len(shifts))) // 2, dtype=torch.int16, device=dev)
    sh = np.array(shifts or [0], np.int32)
    ws = torch.empty(int(L.ss_build_workspace_bytes(W, H)) + 256, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream().cuda_stream

    def ptr(t):
        return None if t is None else t.data_ptr()

    def once():
        _native.check(L.ss_build_tables3(img.data_ptr(), W, H, W, ptr(p64), p32.data_ptr(), ptr(hi16), pitch,
                                         ptr(coarse), len(shifts), sh.ctypes.data, ws.data_ptr(), ws.numel(),
                                         stream), "build")

    once()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        once()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    h = {"p32": plane_hash(p32, 12)}
    if p64 is not None:
        h["p64"] = plane_hash(p64, 12)
    if hi16 is not None:
        h["hi16"] = plane_hash(hi16, 12)
    if coarse is not None:
        h["coarse"] = plane_hash(coarse, 3 * len(shifts))
    return ms, h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cases", default="big,small,odd")
    args = ap.parse_args()
    L = _native.lib()
    cases = []
    if "big" in args.cases:
        cases += [(16384, 16384, "hi16"), (4096, 4096, "u32c")]
    if "small" in args.cases:
        cases += [(2048, 2048, "u32c"), (1920, 1080, "u32c"), (512, 512, "u32c")]
    if "odd" in args.cases:
        cases += [(1300, 777, "int64"), (333, 1000, "int64"), (1000, 333, "u32c"), (17, 900, "int64"), (4097, 130, "int64")]
    res = {}
    for i, (W, H, mode) in enumerate(cases):
        ms, h = run_case(L, W, H, mode, args.reps, 1234 + i)
        res[f"{W}x{H}:{mode}"] = {"ms": round(ms, 4), "hash": h}
        print(f"{W}x{H} {mode}: {ms:.4f} ms", file=sys.stderr)
    print(json.dumps({"pass1": os.environ.get("SS_BUILD_PASS1", "direct"), "band_rows": os.environ.get("SS_BAND_ROWS"),
                      "cases": res}))


if __name__ == "__main__":
    main()
