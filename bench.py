"""bench.py -- positions x scales screened per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

One step = one pass of the hot path over one image of the workload: the 12
integral planes (K1/K2), then for every ladder size the screen (K3), the
survivor list (K4) and the footprint union (K5), then the region popcount.
Inputs are resident in HBM for ``value``; ``e2e`` is the same metric through
the public drop-in ``screen()`` with host numpy in / host results out.

Multi-GPU (torchrun): every rank screens its own image of the workload
(seed + rank) -- per-GPU work fixed, ``scaling: weak``; the only collective
is an NCCL all-gather of the per-rank survivor counts and timings.

``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, the "port"; the reference itself is pure NumPy and not installed
on the GPU box) with every host thread, on the same workload and metric.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate positions x scales screened/sec"
UNIT = "positions*scales/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1, help="BASELINE.json config index (default: configs[1])")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", type=int, default=1, help="capture each step in a CUDA graph")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


POOL_ENGINES = int(os.environ.get("SS_POOL_ENGINES", "4"))  # engines screening a batch's images concurrently


BAND_CONFIGS = (2, 4)  # BASELINE.json: one large image, row bands with halo across GPUs


class BandRunner:
    """One rank's row band (engine with a band frame) behind EnginePool's interface."""

    def __init__(self, engine):
        self.engines = [engine]

    def __len__(self):
        return 1

    def run(self, imgs, tps, **kw):
        self.engines[0].run(imgs[0], tps[0], region=False, **kw)


def workload_config(cfg_idx):
    import workloads as WL

    return WL.CONFIGS[cfg_idx]


def config_json(wl, ladder, n_gpus, extra=None):
    d = {
        "workload": f"BASELINE config {wl.index}: {wl.images} x {wl.width}x{wl.height} u8, template n={wl.template_side}, "
                    f"{len(ladder)} ladder sizes {ladder[0]}..{ladder[-1]}",
        "image": f"{wl.width}x{wl.height}",
        "template_side": wl.template_side,
        "ladder": list(ladder),
        "alpha": wl.alpha,
        "beta": wl.beta,
        "ladder_ratio": wl.ladder_ratio,
        "quantizer": list(wl.q),
        "parallelism": f"image-parallel x{n_gpus}" if n_gpus > 1 else "single GPU",
        "l2": "flushed (256 MiB write) between timed steps; tables are 12 planes (32-bit cells mod 2^32 where exact, else int64) "
              f"({12 * 8 * (wl.width + 1) * (wl.height + 1) / 1e6:.0f} MB) > 126 MB L2",
    }
    if extra:
        d.update(extra)
    return d


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index=0, period=0.05):
        self.samples = []
        self.reasons = set()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # pragma: no cover - no NVML
            self.max_sm = None
        self.period = period
        self._stop = threading.Event()
        self._t = None

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_sm, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_baseline(wl, case, nthreads, max_seconds=30.0):
    """The oracle port (reference algorithm in C, all host threads) on the
    same image and template; the whole ladder, tables included, as the
    reference's screen() does.  Bounded: configs >1 use a row band."""
    import oracle as O

    cfg = O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio, quantizer=O.Quantizer(*wl.q))
    img = case.image
    sample = f"full {wl.width}x{wl.height} image, all {len(O.ladder_sizes(wl.template_side, cfg))} sizes"
    if wl.width * wl.height > 2048 * 2048:
        rows = max(1024, int(2048 * 2048 / wl.width))
        y0 = (wl.height - rows) // 2
        img = np.ascontiguousarray(img[y0:y0 + rows])
        sample = f"{wl.width}x{rows} row band of the image, all sizes"
    t0 = time.perf_counter()
    res = O.screen(img, case.template, cfg, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return {"value": res.patches_tested / dt, "unit": UNIT, "cores": nthreads, "kind": "port",
            "sample": sample + f" (oracle/oracle.c, {res.patches_tested} positions in {dt:.2f} s)",
            "positions": res.patches_tested, "seconds": dt, "result": res, "image": img}


def parity_vs_oracle(cpu, case, wl, dev):
    """The public screen() on the image the CPU baseline screened, against the
    oracle's result: per-size mask bits that differ (the north star's
    threshold-band count; 0 expected: the fp64 path is bit-exact), candidate
    list and stats equality."""
    from paper_1707_05647_b200 import screen
    import workloads as WL

    ref, img = cpu["result"], cpu["image"]
    got = screen(img, case.template, WL.screening_config(wl), device=dev)
    diff = {}
    for m in ref.ladder:
        want = np.packbits(ref.size_masks[m], axis=1, bitorder="little")
        have = got.size_masks.packed(m).view(np.uint8)[:, : want.shape[1]]
        n = int(np.unpackbits(np.bitwise_xor(want, have)).sum())
        if n:
            diff[int(m)] = n
    cand = np.array(ref.candidates, np.int32).reshape(-1, 3)
    return {"image": f"{img.shape[1]}x{img.shape[0]}", "sizes": len(ref.ladder),
            "mask_bit_disagreements": sum(diff.values()), "per_size": diff,
            "candidates_identical": bool(np.array_equal(got.candidates.array(), cand)),
            "stats_identical": (got.stats.patches_tested, got.stats.patches_kept, got.stats.region_pixels_kept) ==
                               (ref.patches_tested, len(ref.candidates), int(ref.region_mask.sum()))}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    import workloads as WL

    wl = workload_config(args.config)
    case = WL.make_cases(wl, images=1)[0]
    nthreads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(wl, case, nthreads)
        if i >= args.warmup:
            vals.append(r)
    pos = sum(r["positions"] for r in vals)
    secs = sum(r["seconds"] for r in vals)
    v = pos / secs
    from paper_1707_05647_b200.config import ladder_sizes
    import workloads as WLm

    ladder = ladder_sizes(wl.template_side, WLm.screening_config(wl))
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(vals), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "impl": "reference",
        "config": config_json(wl, ladder, args.gpus, {"sample": vals[0]["sample"]}),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port", "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def k3_traffic(name, images=1):
    """DRAM bytes (read + write) of the K3 kernels per step of `images`
    images, from the committed ncu launch list of this workload
    (profiles/r1/k3_traffic.json, recorded over rec["images"] images), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1", "k3_traffic.json")
    try:
        with open(path) as f:
            rec = json.load(f).get(name)
    except (OSError, ValueError):
        return None, None
    if not rec:
        return None, None
    return rec["dram_bytes_per_step"] / rec.get("images", 1) * images, rec["source"]


def run_ours(args):
    import torch
    import torch.distributed as dist

    import workloads as WL
    from paper_1707_05647_b200 import _native, screen, screen_batch
    from paper_1707_05647_b200.engine import Engine, EnginePool, prepare_template
    from paper_1707_05647_b200.sharding import plan_bands, screen_sharded

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    wl = workload_config(args.config)
    cfg = WL.screening_config(wl)
    # Single-image configs: every rank screens its own image (weak scaling).
    # Batch configs (config 3: 64 images): a step is the whole batch, images
    # dealt to ranks round-robin (strong scaling), each rank's share screened
    # by an engine pool whose engines overlap on the GPU.
    # Row-band configs (2 and 4) on N > 1 GPUs: one image, rank r decides row
    # band r over tables of its halo'd band (sharding.py; strong scaling);
    # the kept region needs the neighbours' survivors, so it is not part of
    # a band's step (screen_sharded computes it after the gather, in e2e).
    batch = wl.images > 1
    banded = wl.index in BAND_CONFIGS and (world > 1 or os.environ.get("SS_BENCH_BANDS") == "1")
    if banded and not dist.is_initialized():  # SS_BENCH_BANDS=1 on one GPU: the band path with a group of 1
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1,
                                device_id=dev)
    idx = [i for i in range(wl.images) if i % world == rank] if batch else [0 if banded else rank]
    cases = [WL.make_cases(wl, images=1, first_image=i)[0] for i in idx]
    case = cases[0]
    tps = [prepare_template(c.template, cfg, dev) for c in cases]
    tp = tps[0]
    band = plan_bands(wl.height, world, tp.ladder)[rank] if banded else None
    if banded:
        imgs_dev = [torch.from_numpy(np.ascontiguousarray(case.image[band.y_origin:band.y_origin + band.rows])).to(dev)]
        pool = BandRunner(Engine(wl.width, wl.height, dev, band=(band.y_origin, band.rows, band.y_begin, band.y_end)))
    else:
        imgs_dev = [torch.from_numpy(c.image).to(dev) for c in cases]
        pool = EnginePool(wl.width, wl.height, dev, n=min(POOL_ENGINES, len(cases)))
    eng = pool.engines[0]
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    # ── instrumented pass (not timed): cascade stage counts for the roofline ──
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    for e in pool.engines:
        e.stage_counts = counts
    with torch.cuda.stream(stream):
        pool.run(imgs_dev, tps)
    torch.cuda.synchronize()
    stage = counts.cpu().tolist()
    for e in pool.engines:
        e.stage_counts = None
    positions = sum(eng.tested(t) for t in tps)
    survivors = int(stage[3])
    capacity = max(max(1, survivors // len(cases)) * 4, 1 << 16)

    # per-launch events around every screen kernel (dominant kernel)
    ev_pairs = []

    def before(st):  # st: the stream the engine enqueues K3 on
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ev_pairs.append([e, None])

    def after(st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ev_pairs[-1][1] = e

    def step():
        pool.run(imgs_dev, tps, capacity=capacity)

    graph = None
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        if args.graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step()
            graph.replay()
    torch.cuda.synchronize()

    # ── timed region: K steps, L2 flushed between steps (outside the events) ──
    n0 = _native.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index or 0) as clocks:
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.fill_(i & 0xFF)
                starts[i].record(stream)
                if graph is not None:
                    graph.replay()
                else:
                    step()
                ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    n_launch_graph = None
    if graph is None:
        launches = _native.launch_count() - n0
    else:
        # graph replays do not pass through the library: count the launches of one captured step
        n1 = _native.launch_count()
        with torch.cuda.stream(stream):
            step()
        torch.cuda.synchronize()
        n_launch_graph = _native.launch_count() - n1
        launches = n_launch_graph * args.steps
    total_ms = sum(step_ms)

    # per-kernel timing of the screen launches (dominant kernel): one engine,
    # one image at a time (a batch's engines overlap, so their K3 intervals
    # would not add up), scaled to the step's images
    eng.hooks = (before, after)
    with torch.cuda.stream(stream):
        for i in range(3):
            flush.fill_(i)
            eng.run(imgs_dev[0], tps[0], capacity=capacity)
    torch.cuda.synchronize()
    eng.hooks = None
    screen_ms = sum(a.elapsed_time(b) for a, b in ev_pairs) / 3.0 * len(cases)  # per step, all sizes and images

    # max over ranks
    t = torch.tensor([total_ms, float(positions), float(survivors)], dtype=torch.float64, device=dev)
    if world > 1:
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        allt = torch.stack(gathered).cpu().numpy()
        max_ms = float(allt[:, 0].max())
        total_positions = float(allt[:, 1].sum())
    else:
        max_ms = total_ms
        total_positions = float(positions)
    value = total_positions * args.steps / (max_ms / 1e3)

    # ── roofline of the dominant kernel (K3 screen) ──
    peak, peak_src = measured_peak_hbm()
    # algorithmic bytes: SURVEY.md 8(d)'s per-unit figure -- the 12 planes
    # read once per ladder size for ring 0, + 1/8 B of mask bit per position
    # -- with this layout's cell width: 12 x 4 B for sizes screened from the
    # 32-bit planes, 12 x 8 B (SURVEY's 96 B) for sizes that need int64.
    # SURVEY's literal 96 B figure and the cascade-aware count (3 PLAIN planes
    # for every ring-0 evaluation, the other 9 only for mean-projection
    # passers) are reported beside it.
    per_size = [c * len(cases) for c in eng.tested_per_size(tp)]  # the batch's images share the ladder
    alg_bytes = sum(cnt * (12 * (4 if sp.fits32 else 8) + 0.125) for sp, cnt in zip(tp.sizes, per_size))
    achieved = alg_bytes / (screen_ms / 1e3) / 1e9
    cell_bytes = 12 * 8.0 * sum(cnt for sp, cnt in zip(tp.sizes, per_size) if not sp.fits32) / max(positions, 1) + \
        12 * 4.0 * sum(cnt for sp, cnt in zip(tp.sizes, per_size) if sp.fits32) / max(positions, 1)
    cascade_bytes = 24.0 * stage[0] + 72.0 * stage[1] + positions / 8.0
    traffic, traffic_src = k3_traffic(wl.name, len(cases))
    # the 12 planes read exactly once per step (32-bit cells, + int64 cells when a size needs them)
    plane_once = len(cases) * (int(eng.L.ss_tables32_bytes(eng.W, eng.rows)) +
                               (int(eng.L.ss_tables_bytes(eng.W, eng.rows)) if eng.needs_int64(tp) else 0))
    roofline = {
        "bound": "hbm",
        "kernel": ("screen (K3: fused ladder -- ladder_border + ladder_stage1 + ladder_rings kernels -- or, with "
                   "SS_FUSED=0, stage1_kernel + rings_kernel per size; all ladder sizes of one step)"),
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "traffic_source": traffic_src,
        "peak_source": peak_src,
        "alg_bytes_per_step": alg_bytes, "alg_bytes_per_position": alg_bytes / max(positions, 1),
        "plane_bytes_per_position": cell_bytes,
        "survey_96B_bytes_per_step": 96.125 * positions,
        "survey_96B_equiv_GBps": 96.125 * positions / (screen_ms / 1e3) / 1e9,
        "cascade_alg_bytes_per_step": cascade_bytes,
        "cascade_achieved_GBps": cascade_bytes / (screen_ms / 1e3) / 1e9,
        "cascade": {"ring0_evals": stage[0], "ring0_mean_pass": stage[1], "ring0_pass": stage[2],
                    "survivors": stage[3]},
        "screen_ms_per_step": screen_ms, "screen_share_of_step": screen_ms / (total_ms / args.steps),
        "frac_note": ("achieved = SURVEY 8(d)'s algorithmic bytes (every plane read once per ladder size) / K3 time; "
                      "the fused ladder reads each plane about once per row band for all sizes, so frac can exceed 1; "
                      "dram_GBps / dram_frac are the measured K3 DRAM traffic over the same time"),
        "plane_once_bytes_per_step": plane_once,
        "dram_GBps": (traffic / (screen_ms / 1e3) / 1e9) if traffic else None,
        "dram_frac": (traffic / (screen_ms / 1e3) / 1e9 / peak) if traffic else None,
    }
    if batch:
        roofline["screen_ms_note"] = ("batch: one image's K3 time (one engine, nothing overlapping) x the step's "
                                      "images; in the step the pool's engines overlap")

    # ── e2e through the public API (host numpy in, host result out) ──
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        images = [c.image for c in cases]
        templates = [c.template for c in cases]

        def call():
            if batch:
                res = screen_batch(images, templates, cfg, device=dev, engines=POOL_ENGINES)
            elif banded:
                res = [screen_sharded(case.image, case.template, cfg, device=dev)]
            else:
                res = [screen(case.image, case.template, cfg, device=dev)]
            return sum(len(r.candidates.array()) for r in res)  # the survivor lists read back to the host

        for _ in range(3):
            call()
        times = []
        for _ in range(max(5, min(args.steps, 20)) if not batch else 5):
            t0 = time.perf_counter()
            n_cand = call()
            times.append(time.perf_counter() - t0)
        n_inst = sum(math.ceil(m * wl.ladder_ratio) - m + 1 for m in tp.ladder if m >= 8)
        h2d = len(cases) * (case.image.nbytes + case.template.nbytes + n_inst * 36 * 4
                            + sum(sp.blob.nbytes for sp in tp.sizes if sp.blob is not None))
        d2h = n_cand * 12 + len(cases) * (16 + n_inst * 16 * 3 * 8)
        e2e_t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e = {"value": total_positions / float(e2e_t.item()), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * float(e2e_t.item()),
               "ms_min_median_max": [1e3 * min(times), 1e3 * statistics.median(times), 1e3 * max(times)],
               "calls": len(times),
               "api": ("paper_1707_05647_b200.screen_batch(64 numpy images, templates, cfg)" if batch else
                       "paper_1707_05647_b200.sharding.screen_sharded(numpy image, numpy template, cfg) over "
                       f"{world} ranks" if banded else
                       "paper_1707_05647_b200.screen(numpy image, numpy template, cfg)")
                      + " + candidates read back; template feature sets included; masks stay on the device until "
                        "accessed"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        full = cpu_baseline(wl, case, os.cpu_count() or 1)
        parity = parity_vs_oracle(full, case, wl, dev)
        cpu = {k: full[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (batch or banded) else "weak", "vs_baseline": None, "dtype": "int64+f64",
            "data": "synthetic (seeded noise + shapes, SURVEY.md 8(d); template per reference protocol)",
            "config": config_json(wl, tp.ladder, world, {
                "positions_per_step_per_gpu": positions, "survivors_per_step": survivors,
                "per_rank_images": len(cases), "engines": len(pool),
                "row_band": None if band is None else {"y_begin": band.y_begin, "y_end": band.y_end,
                                                       "table_rows": band.rows},
                "cuda_graph": bool(graph is not None)}),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity_vs_oracle": parity,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        }
        print(json.dumps(line))
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
