"""bench.py -- positions x scales screened per second on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Default workload: BASELINE.json config 4 (one 16384^2 u8 image, n = 128, 33
ladder sizes 512..32) -- the largest configuration that fits one B200, and
the one north_star scales over 8 GPUs.  ``--config C`` selects another.

One step = one pass of the hot path over one image (config 3: the 64-image
batch): the 12 integral planes (K1/K2), every ladder size's screen (K3), the
survivor list (K4), the kept region (K5) and its popcount.  ``value`` is
timed with CUDA events on the launching stream over K steps with the inputs
resident in HBM (tables of config 4 are 25.8 GB >> the 126 MB L2; a 256 MiB
write flushes L2 between steps anyway).  ``e2e`` is the same metric through
the public drop-in ``screen()`` with host numpy in and every result array
out: the survivor rows, the packed per-size masks and the packed region.

Multi-GPU (torchrun): configs 2 and 4 are row-banded (sharding.py; strong
scaling): the timed step is the whole sharded screen -- band tables and
screen, the neighbour halo exchange of mask rows, the band's region rows,
the all-gather of counts and survivor rows.  Config 3 deals images to ranks
(strong); configs 0 and 1 run one image per rank (weak).

``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, the "port": the reference is pure NumPy and is not installed on the
GPU box) with every host thread on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate positions x scales screened/sec"
UNIT = "positions*scales/s"
DTYPE = ("u32 planes (cells mod 2^32) + u16 hi planes (cells mod 2^48 for sizes whose sums pass 32 bits) + u16 "
         "coarse bit slices (stage 1); fp32 cell estimates with the fp64 sequence near a boundary")
DEFAULT_CONFIG = 4
BAND_CONFIGS = (2, 4)  # BASELINE.json: one large image, row bands with halo across GPUs
POOL_ENGINES = int(os.environ.get("SS_POOL_ENGINES", "6"))  # sessions screening a batch's images concurrently (measured: 6 beats 2, 4, 8)
L2_BYTES_PER_CLK = 6300  # chip-wide L2 slice throughput cap (B300_MICROARCH.md)
ISSUE_PER_CLK = 4  # warp instructions issued per SM per clock (4 SMSPs)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, help="BASELINE.json config index")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", type=int, default=1, help="capture each step in a CUDA graph (N=1)")
    ap.add_argument("--profile", action="store_true",
                    help="only the warm-up and timed steps (for ncu launch lists: warmup + steps runs), no JSON")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(cfg_idx):
    import workloads as WL

    return WL.CONFIGS[cfg_idx]


def parallelism(wl, n_gpus):
    if n_gpus == 1:
        return "single GPU"
    if wl.index in BAND_CONFIGS:
        return f"row bands x{n_gpus} (halo = largest size's margins)"
    if wl.images > 1:
        return f"images dealt to ranks x{n_gpus}"
    return f"one image per rank x{n_gpus}"


def config_json(wl, ladder, n_gpus):
    """The workload description -- identical in both arms (--impl ours / reference)."""
    return {
        "workload": f"BASELINE config {wl.index}: {wl.images} x {wl.width}x{wl.height} u8 "
                    f"(sigma {wl.sigma:g}, noise {wl.noise:g}), template n={wl.template_side}, "
                    f"{len(ladder)} ladder sizes {ladder[0]}..{ladder[-1]}",
        "image": f"{wl.width}x{wl.height}",
        "images": wl.images,
        "template_side": wl.template_side,
        "ladder": list(ladder),
        "alpha": wl.alpha,
        "beta": wl.beta,
        "ladder_ratio": wl.ladder_ratio,
        "quantizer": list(wl.q),
        "parallelism": parallelism(wl, n_gpus),
        "l2": "inputs larger than L2 (12 planes of (W+1)x(H+1) cells) and a 256 MiB write between timed steps",
    }


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.005):
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

    def _sample(self):
        nv = self.nv
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self._NAMES.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ── CPU samples of the workload (the oracle port; bounded) ──────────────────
# Configs 0, 1 and 3 (one image) run whole; the row-banded configs 2 and 4 run
# a centred core tile with its halo (the core's decisions
# equal the full image's), sized to ~10-30 s of single-core work.
TILE_ALL = {2: (1024, 1024), 4: (1024, 2048)}  # (rows, cols) of the core: all-core leg / reference arm
TILE_ONE = {2: (512, 768), 4: (512, 768)}  # single-core leg


def sample_region(wl, tile):
    if wl.index not in tile:
        return None
    rows, cols = tile[wl.index]
    y0 = (wl.height - rows) // 2
    x0 = (wl.width - cols) // 2
    return (y0, y0 + rows, x0, x0 + cols)


def oracle_cfg(wl):
    import oracle as O

    return O.ScreeningConfig(alpha=wl.alpha, beta=wl.beta, ladder_ratio=wl.ladder_ratio, quantizer=O.Quantizer(*wl.q))


def cpu_sample(wl, case, nthreads, tile, band=False):
    """The oracle port (reference algorithm in C; its scan on `nthreads`
    threads, the rest single-threaded) over the sample: tables, feature sets
    and every ladder size, as the reference's screen() does."""
    import oracle as O

    region = sample_region(wl, tile)
    cfg = oracle_cfg(wl)
    if region is None:
        t0 = time.perf_counter()
        res = O.screen(case.image, case.template, cfg, nthreads=nthreads, band=band)
        dt = time.perf_counter() - t0
        sample = f"full {wl.width}x{wl.height} image, all {len(res.ladder)} sizes"
        return {"positions": res.patches_tested, "seconds": dt, "sample": sample, "result": res, "region": None}
    y0, y1, x0, x1 = region
    t0 = time.perf_counter()
    res = O.screen_tile(case.image, case.template, cfg, y0, y1, x0, x1, nthreads=nthreads, band=band)
    dt = time.perf_counter() - t0
    sample = (f"{x1 - x0}x{y1 - y0} core tile at ({x0}, {y0}) with its halo, all {len(res.ladder)} sizes "
              f"(SURVEY.md App. B.1)")
    return {"positions": res.patches_tested, "seconds": dt, "sample": sample, "result": res, "region": region}


def cpu_baseline(wl, case):
    """Single-core and all-core legs (SURVEY.md 8(d) / BASELINE.md 2).  The
    all-core leg also records band positions: its result is the checker of
    parity_vs_oracle."""
    cores = host_threads()
    one = cpu_sample(wl, case, 1, TILE_ONE)
    full = cpu_sample(wl, case, cores, TILE_ALL, band=True)
    rate = lambda r: r["positions"] / r["seconds"]  # noqa: E731
    out = {
        "value": rate(full), "unit": UNIT, "cores": cores, "kind": "port",
        "sample": full["sample"] + f" (oracle/oracle.c: {full['positions']} positions in {full['seconds']:.2f} s)",
        "single_core": {"value": rate(one), "unit": UNIT, "cores": 1,
                        "sample": one["sample"] + f" ({one['positions']} positions in {one['seconds']:.2f} s)"},
        "cpu_model": cpu_model(), "cpu_count": os.cpu_count(),
    }
    return out, full


def parity_vs_oracle(full, res, wl):
    """The public screen()'s result vs the oracle's on the CPU sample (whole
    image, or the core tile of App. B.1): per-size mask bits that differ,
    band positions (|t - round(t)| <= 1e-6 max(|t|, 1) for some
    channel of some evaluated ring), disagreements outside the band (must be
    0), candidate list, counts and region equality."""
    from paper_1707_05647_b200.screening import unpack_bits

    ref = full["result"]
    region = full["region"]
    W = res.width
    diff, off_band, band = {}, 0, 0
    if region is None:
        y0, y1, x0, x1 = 0, res.height, 0, W
    else:
        y0, y1, x0, x1 = region
    for m in ref.ladder:
        got = unpack_bits(res.size_masks.packed(m)[y0:y1], W)[:, x0:x1]
        want = ref.size_masks[m]
        b = ref.band_masks.get(m) if ref.band_masks else None
        d = got != want
        nd = int(d.sum())
        if b is not None:
            band += int(b.sum())
            off_band += int((d & ~b).sum())
        else:
            off_band += nd
        if nd:
            diff[int(m)] = nd
    cand = res.candidates.array()
    if region is None:
        want_c = np.array(ref.candidates, np.int32).reshape(-1, 3)
        got_c = cand
        want_reg, got_reg = ref.region_mask, res.region_mask
        tested_ok = res.stats.patches_tested == ref.patches_tested
        counts_ok = (res.stats.patches_kept, res.stats.region_pixels_kept) == (ref.patches_kept, ref.region_pixels_kept)
        where = f"full {W}x{res.height} image"
    else:
        sel = (cand[:, 0] >= x0) & (cand[:, 0] < x1) & (cand[:, 1] >= y0) & (cand[:, 1] < y1)
        got_c, want_c = cand[sel], ref.candidates
        ry0, ry1, rx0, rx1 = ref.region_window
        got_reg = unpack_bits(res.region_packed()[ry0:ry1], W)[:, rx0:rx1]
        want_reg = ref.region
        tested_ok = True  # the tile's own count is checked by the tests; stats are whole-image
        counts_ok = int(sel.sum()) == len(want_c)
        where = f"core tile rows [{y0},{y1}) x cols [{x0},{x1}) of the full-image GPU screen"
    return {"compared": where, "sizes": len(ref.ladder), "positions": int(ref.patches_tested),
            "mask_bit_disagreements": sum(diff.values()), "per_size": diff,
            "band_positions": band, "disagreements_outside_band": off_band,
            "candidates_identical": bool(np.array_equal(got_c, want_c)),
            "region_identical": bool(np.array_equal(got_reg, want_reg)),
            "counts_identical": bool(tested_ok and counts_ok)}


def run_reference(args):
    """The reference arm: the oracle port on every host thread, each step one
    bounded sample of the workload (the all-core leg's sample)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    import workloads as WL
    from paper_1707_05647_b200.config import ladder_sizes

    wl = workload_config(args.config)
    case = WL.make_cases(wl, images=1)[0]
    nthreads = host_threads()
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(wl, case, nthreads, TILE_ALL)
        if i >= args.warmup:
            vals.append(r)
    pos = sum(r["positions"] for r in vals)
    secs = sum(r["seconds"] for r in vals)
    v = pos / secs
    ladder = ladder_sizes(wl.template_side, WL.screening_config(wl))
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / len(vals), "higher_is_better": True,
        "scaling": "strong" if (wl.index in BAND_CONFIGS or wl.images > 1) else "weak", "vs_baseline": None,
        "dtype": "int64 tables + f64 features (reference algorithm)", "data": "synthetic (seeded, SURVEY.md 8(d))",
        "impl": "reference",
        "config": config_json(wl, ladder, args.gpus),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads, "kind": "port", "sample": vals[0]["sample"],
                         "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def k3_counters(name, images=1):
    """Per-step ncu figures of the K3 kernels (border + stage 1 + rings) of
    this workload from the committed launch list: DRAM bytes, warp
    instructions, ncu duration.  {} when none is committed."""
    for rnd in ("r2", "r1"):
        path = os.path.join(ROOT, "profiles", rnd, "k3_traffic.json")
        try:
            with open(path) as f:
                rec = json.load(f).get(name)
        except (OSError, ValueError):
            continue
        if rec:
            k = images / rec.get("images", 1)
            out = {"source": rec["source"], "dram_bytes_per_step": rec["dram_bytes_per_step"] * k}
            if "inst_per_step" in rec:
                out["inst_per_step"] = rec["inst_per_step"] * k
                out["inst_stage1_per_step"] = rec.get("inst_stage1_per_step", 0.0) * k
                out["inst_rings_per_step"] = rec.get("inst_rings_per_step", 0.0) * k
            if "l2_bytes_stage1_per_step" in rec:
                out["l2_bytes_stage1_per_step"] = rec["l2_bytes_stage1_per_step"] * k
                out["ms_under_ncu"] = {f: v * k for f, v in rec.get("ms_per_step_under_ncu", {}).items()}
            return out
    return {}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import workloads as WL
    from paper_1707_05647_b200 import _native, screen, screen_batch
    from paper_1707_05647_b200.engine import Engine, EnginePool, prepare_template
    from paper_1707_05647_b200.sharding import ShardedScreener, screen_sharded

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    wl = workload_config(args.config)
    cfg = WL.screening_config(wl)
    batch = wl.images > 1
    banded = wl.index in BAND_CONFIGS and world > 1
    idx = [i for i in range(wl.images) if i % world == rank] if batch else [0 if banded else rank]
    cases = [WL.make_cases(wl, images=1, first_image=i)[0] for i in idx]
    case = cases[0]
    tps = [prepare_template(c.template, cfg, dev) for c in cases]
    tp = tps[0]
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    sharded = None
    if banded:
        sharded = ShardedScreener(wl.width, wl.height, tp, dev)
        imgs_dev = [sharded.upload_band(case.image)]
        pool = None
        eng = sharded.engine
    else:
        imgs_dev = [torch.from_numpy(c.image).to(dev) for c in cases]
        pool = EnginePool(wl.width, wl.height, dev, n=min(POOL_ENGINES, len(cases)))
        eng = pool.engines[0]
    torch.cuda.synchronize()

    def run_step(capacity=None):
        if sharded is not None:
            sharded.step(imgs_dev[0], tp, capacity=capacity)
        else:
            pool.run(imgs_dev, tps, capacity=capacity)

    if args.profile:  # ncu launch lists: exactly warmup + steps runs of the step, nothing else
        for _ in range(args.warmup + args.steps):
            with torch.cuda.stream(stream):
                run_step(1 << 22)
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    # ── instrumented pass (not timed): cascade stage counts for the roofline ──
    counts = torch.zeros(4, dtype=torch.int64, device=dev)
    engines = [eng] if pool is None else pool.engines
    for e in engines:
        e.stage_counts = counts
    with torch.cuda.stream(stream):
        run_step()
    torch.cuda.synchronize()
    stage = counts.cpu().tolist()
    for e in engines:
        e.stage_counts = None
    positions = sum(eng.tested(t) for t in tps)
    survivors = int(stage[3])
    capacity = max(max(1, survivors // len(cases)) * 4, 1 << 16)
    if sharded is not None:
        sharded.set_capacity(capacity)

    graph = None
    use_graph = bool(args.graph) and sharded is None
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            run_step(capacity)
        if use_graph:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                run_step(capacity)
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
                    run_step(capacity)
                ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    if graph is None:
        launches = _native.launch_count() - n0
    else:  # graph replays do not pass through the library: count one captured step's launches
        n1 = _native.launch_count()
        with torch.cuda.stream(stream):
            run_step(capacity)
        torch.cuda.synchronize()
        launches = (_native.launch_count() - n1) * args.steps
    total_ms = sum(step_ms)

    # per-kernel timing of the screen (K3, the dominant kernels): one engine,
    # one image at a time, CUDA events on the stream K3 is launched on
    ev_pairs = []

    def before(st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ev_pairs.append([e, None])

    def after(st):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ev_pairs[-1][1] = e

    eng.hooks = (before, after)
    with torch.cuda.stream(stream):
        for i in range(3):
            flush.fill_(i)
            eng.run(imgs_dev[0], tps[0], capacity=capacity, region=False)
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

    # ── roofline of the dominant kernels (K3: border + stage 1 + rings) ──
    peak, peak_src = measured_peak_hbm()
    k3_s = screen_ms / 1e3
    survey_bytes = 96.125 * positions  # 12 int64 planes once per size + 1/8 B mask bit
    # compulsory bytes of the fused ladder: every plane read once per step
    # (32-bit cells, + int64 cells when a size needs them), the stage-1 list
    # written and read once (8 B entries), the mask bits written once
    plane_once = len(cases) * (int(eng.L.ss_tables32_bytes(eng.W, eng.rows)) +
                               (int(eng.L.ss_tables_bytes(eng.W, eng.rows)) if eng.built_int64 else 0) +
                               (int(eng.L.ss_tables_hi16_bytes(eng.W, eng.rows)) * 3 // 4 if eng.built_hi16 else 0) +
                               int(eng.L.ss_coarse_bytes(eng.W, eng.rows, len(eng.coarse_shifts))))
    compulsory = plane_once + 2 * 8.0 * stage[1] + positions / 8.0
    ctr = k3_counters(wl.name, len(cases))
    clock_mhz = clocks.summary().get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    issue_slots = ISSUE_PER_CLK * sms * clock_mhz * 1e6 * k3_s
    roofline = {
        "bound": "hbm",
        "kernel": "K3 screen: ladder_border + ladder_stage1 + ladder_rings (all ladder sizes of one step)",
        "achieved": survey_bytes / k3_s / 1e9, "peak": peak, "unit": "GB/s",
        "frac": survey_bytes / k3_s / 1e9 / peak, "traffic": ctr.get("dram_bytes_per_step"),
        "peak_source": peak_src,
        "alg_bytes_per_position": 96.125,
        "alg_bytes_note": ("SURVEY.md 8(d): 12 int64 planes read once per ladder size + 1/8 B of mask bit per "
                           "position*scale; the fused ladder reads the planes about once per row band for all "
                           "sizes, so this frac can exceed 1 and is not HBM efficiency -- see compulsory / dram / "
                           "issue below"),
        "k3_ms_per_step": screen_ms, "k3_share_of_step": screen_ms / (total_ms / args.steps),
        "compulsory": {"bytes_per_step": compulsory, "GBps": compulsory / k3_s / 1e9,
                       "frac": compulsory / k3_s / 1e9 / peak,
                       "what": ("each plane stage 1 and the rings read (u32, hi16 / int64, coarse slices) once per "
                                "step + stage-1 list written and read (8 B entries) + mask bits")},
        "dram": ({"bytes_per_step": ctr["dram_bytes_per_step"], "GBps": ctr["dram_bytes_per_step"] / k3_s / 1e9,
                  "frac": ctr["dram_bytes_per_step"] / k3_s / 1e9 / peak, "source": ctr["source"]}
                 if ctr else None),
        "issue": ({"warp_inst_per_step": ctr["inst_per_step"], "slots_per_step": issue_slots,
                   "frac": ctr["inst_per_step"] / issue_slots,
                   "warp_inst_per_position_stage1": ctr["inst_stage1_per_step"] / max(positions, 1),
                   "warp_inst_per_rings_candidate": ctr["inst_rings_per_step"] / max(stage[1], 1),
                   "peak": f"{ISSUE_PER_CLK} warp inst/clk x {sms} SMs x {clock_mhz:.0f} MHz",
                   "source": ctr["source"]} if ctr.get("inst_per_step") else None),
        "cascade": {"ring0_evals": stage[0], "ring0_mean_pass": stage[1], "ring0_pass": stage[2],
                    "survivors": stage[3]},
    }
    # stage 1 moves its corner boxes L2 -> shared memory by TMA and is bound by
    # that path, not by HBM: its L2 bytes (ncu lts__t_bytes) over its ncu time
    # against the L2 slices' cap (B300_MICROARCH.md: ~6300 B/clk chip-wide)
    s1_ms = (ctr.get("ms_under_ncu") or {}).get("stage1")
    if s1_ms and ctr.get("l2_bytes_stage1_per_step"):
        l2_peak = L2_BYTES_PER_CLK * clock_mhz * 1e6 / 1e9
        roofline["stage1_l2"] = {
            "bound": "l2", "bytes_per_step": ctr["l2_bytes_stage1_per_step"], "ms_per_step_under_ncu": s1_ms,
            "achieved": ctr["l2_bytes_stage1_per_step"] / (s1_ms / 1e3) / 1e9, "peak": l2_peak, "unit": "GB/s",
            "frac": ctr["l2_bytes_stage1_per_step"] / (s1_ms / 1e3) / 1e9 / l2_peak,
            "peak_source": f"{L2_BYTES_PER_CLK} B/clk (B300_MICROARCH.md, LTS throughput cap) x {clock_mhz:.0f} MHz",
            "source": ctr["source"]}
        roofline["ms_under_ncu"] = ctr["ms_under_ncu"]

    # ── e2e through the public API (host numpy in, every result array out) ──
    e2e = None
    last = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        # the inputs live in pinned host memory (the contract's e2e: each step
        # copies them host -> device); the API takes them as numpy arrays

        def pinned(a):
            t = torch.empty(a.shape, dtype=torch.uint8, pin_memory=True)
            t.numpy()[...] = a
            return t.numpy()

        images = [pinned(c.image) for c in cases]
        templates = [pinned(c.template) for c in cases]
        d2h = [0]

        def call():
            if batch:
                res = screen_batch(images, templates, cfg, device=dev, engines=POOL_ENGINES)
            elif banded:
                res = [screen_sharded(images[0], templates[0], cfg, device=dev)]
            else:
                res = [screen(images[0], templates[0], cfg, device=dev)]
            nbytes = 0
            for r in res:  # survivor rows, packed masks of every size, packed region -> host
                nbytes += r.candidates.array().nbytes + r.size_masks.packed_all().nbytes + r.region_packed().nbytes
            d2h[0] = nbytes
            return res

        for _ in range(2):
            last = call()
        times = []
        for _ in range(max(5, min(args.steps, 10)) if not batch else 3):
            t0 = time.perf_counter()
            last = call()
            times.append(time.perf_counter() - t0)
        n_inst = sum(math.ceil(m * wl.ladder_ratio) - m + 1 for m in tp.ladder if m >= 8)
        h2d = len(cases) * (case.image.nbytes + case.template.nbytes + n_inst * 36 * 4
                            + sum(sp.blob.nbytes for sp in tp.sizes if sp.blob is not None))
        e2e_t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        e2e_s = float(e2e_t.cpu())
        e2e = {"value": total_positions / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h[0]), "ms_per_step": 1e3 * e2e_s,
               "ms_min_median_max": [1e3 * min(times), 1e3 * statistics.median(times), 1e3 * max(times)],
               "calls": len(times),
               "inputs": "numpy arrays over pinned host memory",
               "api": ("paper_1707_05647_b200.screen_batch(64 numpy images, templates, cfg)" if batch else
                       f"paper_1707_05647_b200.sharding.screen_sharded(numpy image, template, cfg) over {world} ranks"
                       if banded else "paper_1707_05647_b200.screen(numpy image, numpy template, cfg)")
                      + "; then candidates.array(), size_masks.packed_all(), region_packed() to the host; "
                        "template feature sets included"}

    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu, full = cpu_baseline(wl, case)
        if last is None:
            last = [screen(case.image, case.template, cfg, device=dev)]
        parity = parity_vs_oracle(full, last[0], wl)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if (batch or wl.index in BAND_CONFIGS) else "weak", "vs_baseline": None,
            "dtype": DTYPE,
            "data": "synthetic (seeded noise + shapes, SURVEY.md 8(d); template per reference protocol)",
            "config": config_json(wl, tp.ladder, world),
            "run": {"positions_per_step": total_positions, "positions_per_step_rank0": positions,
                    "survivors_per_step_rank0": survivors, "images_rank0": len(cases),
                    "engines": 1 if pool is None else len(pool), "cuda_graph": graph is not None,
                    "row_band_rank0": None if sharded is None else vars(sharded.band)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity_vs_oracle": parity,
            "band_positions": None if parity is None else parity["band_positions"],
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
