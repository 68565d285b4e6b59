#!/usr/bin/env python
"""hfuse-b200 benchmark: the ten horizontally fused DL kernel pairs on B200 (C2/C1/C5).

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl hfuse|reference]
  (N > 1: launched by torch.distributed.run, one rank per GPU, weak scaling)

Workload: every pair of {BatchNorm-stats, Hist, Im2Col, MaxPool, Upsample} at the C2
shapes (paper_2007_01277_b200/pairs.py, 'full' sizes; each pair reads/writes >= 410 MB,
larger than the 126 MB L2, so no flush is needed between steps). Setup (untimed): the
profile-guided split search (search_config on the device backend) picks (d1, regcap)
per pair; the unfused sequential and two-stream baselines are timed per pair.
A step = the ten best-split fused kernels, back to back, inputs resident in HBM.
  value    = us per step (max over ranks), lower is better
  e2e      = us per step through the C ABI with pinned HOST inputs: H2D of each pair's
             inputs + fused launch + D2H of its outputs, all inside the timed region
  roofline = the dominant fused kernel's algorithmic bytes / its mean launch time vs the
             measured HBM copy bandwidth (MEASURED_PEAKS.json)
For N > 1 each rank owns its own batch shard (seed offset = rank) and the step ends with
the single NCCL reduction of the shard outputs (histogram bins all-reduce + BatchNorm
stats all-gather), timed inside the step.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused-pair speedup vs max(sequential, 2-stream) unfused, µs; %roofline at 1/8 B200"
SAMPLE_DIV = 32  # CPU baseline sample = 1/32 of each member's workload (~10-30 s of CPU work per step)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------------------
# CPU reference: the reference interpreter (oracle/_ref) on a bounded sample
# ---------------------------------------------------------------------------------------

def sample_images(div=SAMPLE_DIV):
    """Per-member sample images: 1/div of the full workload along the batch/channel axis."""
    C, n, mp, us, ic = 256 // div, 51380224 // div, 4096 // div, 16384 // div, 2048 // div
    return {
        "bn": (f"array bn_x float32 {64 * C * 3136} seed 1 uniform -1 1\narray bn_stats float32 {2 * C} zero\n"
               f"scalar bn_N int32 64\nscalar bn_C int32 {C}\nscalar bn_HW int32 3136\n"),
        "hist": f"array hi_x float32 {n} seed 2 uniform -4 4\narray hi_out int32 64 zero\nscalar hi_n int32 {n}\n",
        "maxpool": (f"array mp_x float32 {mp * 112 * 112} seed 3 uniform -1 1\narray mp_y float32 {mp * 56 * 56} zero\n"
                    f"array mp_idx int32 {mp * 56 * 56} zero\nscalar mp_NC int32 {mp}\nscalar mp_H int32 112\n"
                    "scalar mp_W int32 112\nscalar mp_OH int32 56\nscalar mp_OW int32 56\n"),
        "upsample": (f"array us_x float32 {us * 28 * 28} seed 4 uniform -1 1\narray us_y float32 {us * 56 * 56} zero\n"
                     f"scalar us_NC int32 {us}\nscalar us_IH int32 28\nscalar us_IW int32 28\n"
                     "scalar us_OH int32 56\nscalar us_OW int32 56\n"),
        "im2col": (f"array ic_x float32 {ic * 56 * 56} seed 5 uniform -1 1\narray ic_col float32 {ic * 9 * 56 * 56} zero\n"
                   f"scalar ic_NC int32 {ic}\nscalar ic_H int32 56\nscalar ic_W int32 56\n"),
    }


def cpu_reference_step(pairs_mod, workdir, cores):
    """One step of the reference's CPU execution: `seq` (run_functional k1 then k2,
    exec.cpp:958-965) of the naive member kernels for all ten pairs on the sample, the pairs
    spread over `cores` processes. Returns (wall seconds, kind, sample description)."""
    from oracle import oracle
    imgs = sample_images()
    jobs = []
    for a, b in pairs_mod.PAIRS:
        ia = os.path.join(workdir, f"{a}.img")
        ib = os.path.join(workdir, f"{b}.img")
        for k, p in ((a, ia), (b, ib)):
            if not os.path.exists(p):
                with open(p, "w") as f:
                    f.write(imgs[k])
        ka = os.path.join(pairs_mod.KERNELS, "ref", pairs_mod.MEMBERS[a].stem + ".mk")
        kb = os.path.join(pairs_mod.KERNELS, "ref", pairs_mod.MEMBERS[b].stem + ".mk")
        if oracle.have_ref():
            jobs.append([oracle.REF, "seq", ka, kb, "--mem", ia, "--mem", ib, "--grid", "2"])
    if not jobs:
        return None
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=cores) as pool:
        codes = list(pool.map(lambda c: subprocess.run(c, stdout=subprocess.DEVNULL,
                                                        stderr=subprocess.DEVNULL).returncode, jobs))
    if any(codes):
        raise RuntimeError(f"reference interpreter failed: {codes}")
    wall = time.perf_counter() - t0
    return wall


def cpu_baseline(pairs_mod, steps=1):
    from oracle import oracle
    cores = min(len(pairs_mod.PAIRS), os.cpu_count() or 1)
    with tempfile.TemporaryDirectory() as d:
        if oracle.have_ref():
            walls = [cpu_reference_step(pairs_mod, d, cores) for _ in range(steps)]
            wall = statistics.median(walls)
            return {"value": wall * SAMPLE_DIV * 1e6, "unit": "us", "cores": cores, "kind": "reference",
                    "sample": f"reference interpreter (oracle/_ref mkfuse_ref seq, run_functional) on 1/{SAMPLE_DIV} "
                              f"of every member's workload for all 10 naive pairs, {cores} pairs in parallel, "
                              f"wall {wall:.2f} s x {SAMPLE_DIV}"}
        # port: the C restatement, multi-threaded
        import numpy as np
        t0 = time.perf_counter()
        n = 51380224 // SAMPLE_DIV
        x = oracle.fill_uniform(n, 1, -1.0, 1.0)
        for _ in range(4):
            oracle.bn_stats(x, 64, 256 // SAMPLE_DIV, 3136)
            oracle.hist(x)
            oracle.maxpool(x, 4096 // SAMPLE_DIV, 112, 112)
            oracle.upsample(x[:n // 4], 16384 // SAMPLE_DIV, 28, 28)
            oracle.im2col(x[:n // 8], 2048 // SAMPLE_DIV, 56, 56)
        wall = time.perf_counter() - t0
        del np
        return {"value": wall * SAMPLE_DIV * 1e6, "unit": "us", "cores": oracle.threads(), "kind": "port",
                "sample": f"C restatement on 1/{SAMPLE_DIV} of every member x 4 pair-appearances"}


_COLL = {}


def _install_collectives(dist, backend):
    """all_reduce / all_gather on CUDA tensors: NCCL directly; other backends (the one-GPU
    gloo validation of the multi-rank path) stage through host memory."""
    _COLL["dist"], _COLL["backend"] = dist, backend


def all_reduce(t, op="sum"):
    dist = _COLL["dist"]
    o = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}[op]
    if _COLL["backend"] == "nccl":
        dist.all_reduce(t, op=o)
        return t
    c = t.cpu()
    dist.all_reduce(c, op=o)
    t.copy_(c)
    return t


def all_gather(t, world):
    import torch
    dist = _COLL["dist"]
    if _COLL["backend"] == "nccl":
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return parts
    c = t.cpu()
    parts = [torch.empty_like(c) for _ in range(world)]
    dist.all_gather(parts, c)
    return [p.to(t.device) for p in parts]


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2007_01277_b200 import pairs as pairs_mod
    from oracle import oracle
    cores = min(len(pairs_mod.PAIRS), os.cpu_count() or 1)
    if not oracle.have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/mkfuse_ref not built (needs /root/reference)"}))
        return 0
    with tempfile.TemporaryDirectory() as d:
        for _ in range(args.warmup):
            cpu_reference_step(pairs_mod, d, cores)
        walls = [cpu_reference_step(pairs_mod, d, cores) for _ in range(args.steps)]
    wall = statistics.median(walls)
    # weak scaling: the N-GPU job is N batch shards of this workload; the CPU reference runs
    # them one after another on the same cores (one shard measured, N times its time)
    shards = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    us = wall * SAMPLE_DIV * 1e6 * shards
    line = {
        "metric": METRIC, "impl": "reference", "value": us, "unit": "us", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32/int32", "data": "synthetic (seeded splitmix64)",
        "config": {"workload": "C2: 10 DL pairs (BN, Hist, Im2Col, MaxPool, Upsample), naive member forms, "
                               f"sequential run_functional, extrapolated from a 1/{SAMPLE_DIV} sample",
                   "sample_div": SAMPLE_DIV},
        "cpu_baseline": {"value": us, "unit": "us", "cores": cores, "kind": "reference",
                         "sample": f"mkfuse_ref seq on 1/{SAMPLE_DIV} of each member, 10 pairs over {cores} processes"
                                   + (f", x {shards} shards (weak scaling)" if shards > 1 else "")},
        "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------

class ClockSampler:
    """SM clocks and throttle reasons sampled every 10 ms through NVML (nvidia-smi's source)
    while the timed region runs (B200_PROFILING.md clocks rule); nvidia-smi as a fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.rows = []  # (sm_mhz, reasons set)
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _nvml_loop(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
        while not self._stop.is_set():
            mhz = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            bits = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((mhz, {name for name, attr in self.REASONS if bits & getattr(N, attr)}))
            self._stop.wait(0.01)

    def _smi_loop(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.max_mhz = float(out[1])
                self.rows.append((float(out[0]), {n for (n, _), v in zip(self.REASONS, out[2:]) if v.strip() == "Active"}))
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        def run():
            try:
                self._nvml_loop()
            except Exception:
                self._smi_loop()
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(set().union(*(r[1] for r in self.rows))), "samples": len(self.rows)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hfuse", choices=["hfuse", "reference"])
    ap.add_argument("--grid", type=int, default=296, help="crypto suite grid (148 SMs x 2 blocks)")
    ap.add_argument("--grids", default="296,592,1184,2368",
                    help="launch grids tried for every DL member and fused pair (multiples of 148 SMs)")
    ap.add_argument("--search-reps", type=int, default=5)
    ap.add_argument("--d0s", default="1024,512", help="fused block sizes searched for the DL pairs")
    ap.add_argument("--shapes", default="conv2", choices=["conv2", "conv3"],
                    help="DL tensor shapes: ResNet-50 conv2_x (the C2 configuration, default) or conv3_x")
    ap.add_argument("--granularity", type=int, default=64,
                    help="split step of the partition sweep (the reference sweeps 128)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pairs", default="all")
    ap.add_argument("--ratios", default="0.5,1,2",
                    help="workload-ratio study: t_b/t_a targets for every DL pair ('none' to skip)")
    ap.add_argument("--no-crypto", action="store_true", help="skip the C3/C4 crypto suite")
    ap.add_argument("--l2", default="steady", choices=["steady", "flush"],
                    help="DL timing protocol: steady = repetitions back to back with every pair's inputs "
                         "> L2, so each repetition also pays the write-back of the previous one's dirty "
                         "lines (the bench contract's inputs-larger-than-L2 option); flush = a read sweep "
                         "before every repetition (drains those write-backs outside the timed region)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HF_BENCH_DIST=gloo: the multi-rank path validated on ONE GPU (ranks share cuda:0, the
    # collectives go through host memory); production runs use NCCL, one rank per GPU
    backend = os.environ.get("HF_BENCH_DIST", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    _install_collectives(dist, backend)
    from paper_2007_01277_b200 import hfuse as hf
    from paper_2007_01277_b200 import pairs as P

    pair_list = P.PAIRS if args.pairs == "all" else [tuple(p.split("+")) for p in args.pairs.split(",")]
    keys = sorted({k for p in pair_list for k in p})
    grids = [int(g) for g in args.grids.split(",")] if args.grids else [args.grid]
    flush = args.l2 == "flush"
    d0s = [int(x) for x in args.d0s.split(",")]
    stream = torch.cuda.current_stream()

    # ---- setup: one image holding every member's arrays (bound by name), per-rank shard seed
    shape = "full" if args.shapes == "conv2" else args.shapes
    img = hf.Image(P.MEMBERS[keys[0]].sizes[shape](rank).image)
    for k in keys[1:]:
        img.merge(hf.Image(P.MEMBERS[k].sizes[shape](rank).image))
    img.upload(stream)
    work = {k: P.MEMBERS[k].sizes[shape](rank) for k in keys}
    src = {k: P.source("b200", P.MEMBERS[k].stem) for k in keys}
    # JIT specialization: every module folds this image's scalar shapes into its code
    unfused = {k: hf.Module.kernel(src[k], grid=grids[0], specialize=img) for k in keys}
    # The members are grid-stride loops, so the launch grid is a free parameter. Every variant
    # gets its own best grid: each unfused member alone (the baselines), each fused pair jointly
    # with its split and register cap (the search is repeated per grid; the compiled candidates
    # are cached, so only the timing repeats).
    mgrid, member_sweep = {}, {}
    for k in keys:
        ts = {g: hf.time("single", unfused[k], None, img, g, warmup=2, reps=10, flush_l2=flush,
                         stream=stream)["iqm_us"]
              for g in grids}
        mgrid[k] = min(ts, key=ts.get)
        member_sweep[k] = {str(g): round(t, 2) for g, t in ts.items()}

    results = []
    fused = {}
    pgrid = {}
    two_grids = {}
    t_setup = time.perf_counter()
    for a, b in pair_list:
        r, grid, trace = None, None, []
        # fused block sizes: 1024 threads (2 blocks / SM) and 512 (4 blocks / SM, twice the
        # grid), each with every split at the search granularity
        for d0 in d0s:
            for g in grids if d0 == 1024 else [2 * x for x in grids]:
                rg = hf.search(src[a], src[b], img, d0=d0, grid=g, reps=args.search_reps, warmup=2,
                               specialize=True, flush_l2=flush, granularity=args.granularity)
                trace += [(d0, g, t["d1"], t["reg_cap"], round(t["us"], 2)) for t in rg["trace"]]
                if r is None or rg["best_time"] < r["best_time"]:
                    r, grid = rg, g
        cap = r["reg_cap"]
        m = hf.Module.fused(src[a], src[b], r["d1"], r["d2"], regcap=cap if cap else "off", grid=grid,
                            specialize=img)
        fused[(a, b)] = m
        pgrid[(a, b)] = grid
        ga, gb = mgrid[a], mgrid[b]
        # one protocol for all variants: L2 flushed (clean) before every repetition
        fz = hf.time("single", m, None, img, grid, warmup=5, reps=60, flush_l2=flush, stream=stream)
        seq = hf.time("sequential", unfused[a], unfused[b], img, ga, gb, warmup=5, reps=60, flush_l2=flush,
                      stream=stream)
        two, tga, tgb = best_two_stream(hf, unfused[a], unfused[b], img, ga, gb, grids, flush, stream)
        two_grids[(a, b)] = (tga, tgb)
        ta = hf.time("single", unfused[a], None, img, ga, warmup=2, reps=10, flush_l2=flush, stream=stream)
        tb = hf.time("single", unfused[b], None, img, gb, warmup=2, reps=10, flush_l2=flush, stream=stream)
        # baselines of the paper's comparison: the reference's naive goto fusion of the naive
        # member forms at the same split, and vertical fusion (VFuse) of the B200 forms
        naive = hf.Module.naive(P.source("ref", P.MEMBERS[a].stem), P.source("ref", P.MEMBERS[b].stem),
                                r["d1"], r["d2"], grid)
        tn = hf.time("single", naive, None, img, grid, warmup=2, reps=10, flush_l2=flush, stream=stream)
        vert = hf.Module.vertical(src[a], src[b], grid, specialize=img)
        tv = min(hf.time("single", vert, None, img, g, warmup=2, reps=10, flush_l2=flush, stream=stream)["iqm_us"]
                 for g in grids)
        results.append({"pair": f"{a}+{b}", "grid": grid, "d0": r["d1"] + r["d2"], "d1": r["d1"], "d2": r["d2"],
                        "reg_cap": cap,
                        "grid_a": ga, "grid_b": gb, "two_stream_grids": [tga, tgb],
                        "bytes": work[a].bytes + work[b].bytes, "regs": m.info.regs,
                        "blocks_per_sm": m.info.blocks_per_sm, "fused_us": fz["iqm_us"],
                        "seq_us": seq["iqm_us"], "two_stream_us": two["iqm_us"],
                        "a_us": ta["iqm_us"], "b_us": tb["iqm_us"],
                        "naive_fused_us": tn["iqm_us"], "vertical_us": tv,
                        "search_trace": trace})
    stream_ceilings(hf, P, results, work, grids, flush, stream)
    setup_s = time.perf_counter() - t_setup

    import ctypes
    _cudart = ctypes.CDLL("libcudart.so.12")

    def cudart_copy(dst_tensor, src_ptr, nbytes):
        # device-to-device copy of a libhfuse image array into a torch tensor, on the stream
        _cudart.cudaMemcpyAsync(ctypes.c_void_p(dst_tensor.data_ptr()), ctypes.c_void_p(src_ptr),
                                ctypes.c_size_t(nbytes), 3, ctypes.c_void_p(stream.cuda_stream))

    def reduce_outputs():
        # the path's single exchange: histogram bins (int32 sum) + per-rank BN stats gather
        if "hist" in keys:
            bins = torch.empty(64, dtype=torch.int32, device="cuda")
            cudart_copy(bins, img.device_ptr("hi_out"), 64 * 4)
            all_reduce(bins)
        if "bn" in keys:
            st = torch.empty(512, dtype=torch.float32, device="cuda")
            cudart_copy(st, img.device_ptr("bn_stats"), 512 * 4)
            all_gather(st, world)

    # ---- timed region: K steps of the ten fused kernels, back to back on one stream. The pairs
    # are independent, so each fused kernel is a programmatic dependent launch (overlap=True:
    # it may start while its predecessor drains -- the B200's answer to the exposed tail of a
    # one-stream chain). A second pass without overlap and with per-kernel events times each
    # kernel alone inside the step (the roofline's achieved bandwidth).
    def step(record=None, overlap=False):
        for i, (a, b) in enumerate(pair_list):
            if record is not None:
                record[i][0].record(stream)
            fused[(a, b)].run(img, pgrid[(a, b)], stream, overlap=overlap)
            if record is not None:
                record[i][1].record(stream)
        if dist is not None:
            reduce_outputs()

    side = torch.cuda.Stream()

    def unfused_step():
        # the same ten pairs unfused, each pair's two kernels concurrent on two streams (at the
        # pair's best two-stream grids)
        for a, b in pair_list:
            ga, gb = two_grids[(a, b)]
            side.wait_stream(stream)
            unfused[a].run(img, ga, stream)
            unfused[b].run(img, gb, side)
            stream.wait_stream(side)
        if dist is not None:
            reduce_outputs()

    def unfused_overlap_step():
        # the same twenty unfused kernels on one stream, each a programmatic dependent launch
        for a, b in pair_list:
            unfused[a].run(img, mgrid[a], stream, overlap=True)
            unfused[b].run(img, mgrid[b], stream, overlap=True)
        if dist is not None:
            reduce_outputs()

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        e0.record(stream)
        for s in range(args.steps):
            fn(s)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step(overlap=True)
            step()
            unfused_step()
            unfused_overlap_step()
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in pair_list] for _ in range(args.steps)]
        torch.cuda.nvtx.range_push("step")  # ncu --nvtx --nvtx-include "step/": the launch list of `value`
        total_ms = timed(lambda s: step(overlap=True))
        torch.cuda.nvtx.range_pop()
        serial_ms = timed(lambda s: step(ev[s]))
        unfused_ms = timed(lambda s: unfused_step())
        unfused_overlap_ms = timed(lambda s: unfused_overlap_step())
    ms = torch.tensor([total_ms, unfused_ms, unfused_overlap_ms, serial_ms], device="cuda")
    if dist is not None:
        all_reduce(ms, "max")
    us_per_step = ms[0].item() * 1000.0 / args.steps
    unfused_us_per_step = ms[1].item() * 1000.0 / args.steps
    unfused_overlap_us_per_step = ms[2].item() * 1000.0 / args.steps
    serial_us_per_step = ms[3].item() * 1000.0 / args.steps

    hbm_peak, peak_src = load_peaks()
    for i, res in enumerate(results):
        ts = [ev[s][i][0].elapsed_time(ev[s][i][1]) * 1000.0 for s in range(args.steps)]
        res["in_step_us"] = statistics.median(ts)
        res["in_step_us_mean"] = statistics.mean(ts)
        base = min(res["seq_us"], res["two_stream_us"])
        res["speedup"] = base / res["fused_us"]
        res["roofline_us"] = res["bytes"] / (hbm_peak * 1e3)
        res["roofline_frac"] = res["roofline_us"] / res["fused_us"]
    geo = 1.0
    for res in results:
        geo *= res["speedup"]
    geo **= 1.0 / len(results)
    dom = max(results, key=lambda r: r["in_step_us_mean"])
    achieved = dom["bytes"] / (dom["in_step_us_mean"] * 1e3)  # GB/s, mean launch time inside the step

    # ---- e2e: the same step through the C ABI from pinned host buffers
    e2e = e2e_step(hf, torch, P, pair_list, fused, work, keys, pgrid, stream, args)
    if dist is not None:  # the job's end-to-end step ends with its slowest rank
        t = torch.tensor([e2e["value"]], device="cuda", dtype=torch.float64)
        all_reduce(t, "max")
        e2e["value"] = t.item()
        e2e["h2d_bytes_per_step"] *= world
        e2e["d2h_bytes_per_step"] *= world
    del img  # free the DL images before the crypto suite (the Ethash DAG alone is 4 GiB)
    ratio_res = None
    if world == 1 and args.ratios != "none":  # a one-GPU study (C2); shards run only the step
        member_us = {k: min(v.values()) for k, v in member_sweep.items()}
        ratio_res = ratio_study(hf, P, pair_list, src, shape, rank, grids, d0s, flush, stream, member_us, args)
    crypto_res = None
    clk = clocks.summary()
    if not args.no_crypto:
        crypto_res = crypto_suite(hf, torch, args, rank, world, stream, sm_mhz=clk.get("sm_mhz"),
                                  hbm_peak=hbm_peak)

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            # ncu dram__bytes_read.sum + dram__bytes_write.sum of this fused kernel, one launch
            # (scripts/ncu_members.py under ncu -> scripts/ncu_summarize.py traffic)
            traffic = json.load(open(tpath))[dom["pair"]]["dram_bytes"]
        except Exception:
            traffic = None

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return 0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(P)
        except Exception as e:  # the baseline is reported, not required
            cpu = {"value": None, "unit": "us", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC,
        "value": us_per_step,
        "unit": "us",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": us_per_step / 1000.0,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32/int32",
        "data": "synthetic (splitmix64-seeded in HBM; per-rank shard seed)",
        "config": {"workload": ("C2: all 10 DL pairs of {BatchNorm-stats 64x256x56x56, Hist 64x256x56x56, "
                                "Im2Col 32x64x56x56, MaxPool 64x64x112x112, Upsample 64x256x28x28}"
                                if shape == "full" else
                                "C5 shapes (ResNet-50 conv3_x): all 10 DL pairs of {BatchNorm-stats 64x512x28x28, "
                                "Hist 64x512x28x28, Im2Col 32x128x28x28, MaxPool 64x128x56x56, Upsample 64x512x14x14}")
                               + " fused at the searched best (block size d0 in {1024, 512}, grid, split, register cap)",
                   "grids": grids,
                   "pairs": len(results), "member_grid_us": member_sweep,
                   "l2": ("step: inputs per pair > 126 MB L2, no flush; per-pair tables: "
                          + ("back-to-back repetitions (each pays the previous one's write-back)" if not flush
                             else "read-sweep flush before every repetition")),
                   "parallelism": f"dp{world} (batch shards)"},
        "speedup_geomean": geo,
        "unfused_two_stream_step_us": unfused_us_per_step,
        "unfused_overlap_step_us": unfused_overlap_us_per_step,
        "fused_serial_step_us": serial_us_per_step,
        "step": "ten fused kernels on one stream as programmatic dependent launches (value); "
                "fused_serial: the same without overlap; unfused: each pair on two streams, or all "
                "twenty kernels as programmatic dependent launches on one stream",
        "step_speedup": min(unfused_us_per_step, unfused_overlap_us_per_step) / us_per_step,
        "pairs": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items() if k != "search_trace"}
                  for r in results],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "kernel": f"fused {dom['pair']}",
                     "peak_source": peak_src, "algorithmic_bytes": dom["bytes"]},
        "e2e": e2e,
        "gpu_launches": len(pair_list) * args.steps,
        "clocks": clk,
        "cpu_baseline": cpu,
        "setup_s": round(setup_s, 1),
        "search": {r["pair"]: r["search_trace"] for r in results},
        "ratios": ratio_res,
        "crypto": crypto_res,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


CRYPTO_COUNTS = {"sha256d": 1 << 24, "blake2b": 1 << 23, "blake256": 1 << 24, "ethash": 1 << 20}
ETHASH_PAGES = 1 << 25  # 4 GiB synthetic DAG (>> the 126 MB L2)


def crypto_roofline(nonces, t_us, sm_mhz, hbm_peak):
    """Pair roofline of SURVEY.md §8d: max(issue time, HBM time). Issue time = warp
    instructions / (148 SMs x 4 schedulers x f_sm), with each member's warp instructions per
    nonce measured once by ncu (scripts/ncu_crypto_inst.py -> profiles/crypto_inst.json; SHA-256d
    and the BLAKEs are data-independent, Ethash's page walk is fixed at 64 accesses). HBM time:
    Ethash reads 64 pages x 128 B per nonce. Also the ALU-pipe bound (16 lanes per scheduler:
    2 cycles per warp ALU instruction), the tighter ceiling for the rotate/xor-heavy hashes."""
    path = os.path.join(ROOT, "profiles", "crypto_inst.json")
    if not os.path.exists(path) or not sm_mhz:
        return None
    table = json.load(open(path))
    if any(k not in table for k in nonces):
        return None
    slots = 148 * 4 * sm_mhz * 1e6
    winst = sum(n * table[k]["warp_inst_per_nonce"] for k, n in nonces.items())
    alu = sum(n * table[k]["alu_warp_inst_per_nonce"] for k, n in nonces.items())
    t_issue = winst / slots * 1e6
    t_alu = 2 * alu / slots * 1e6
    t_hbm = sum(n * 64 * 128 for k, n in nonces.items() if k == "ethash") / (hbm_peak * 1e3)
    t_roof = max(t_issue, t_hbm)
    return {"bound": "issue" if t_issue >= t_hbm else "hbm", "roofline_us": t_roof, "frac": t_roof / t_us,
            "issue_us": t_issue, "alu_pipe_us": t_alu, "alu_frac": t_alu / t_us, "hbm_us": t_hbm,
            "warp_inst": winst, "sm_mhz": sm_mhz}


def crypto_suite(hf, torch, args, rank, world, stream, sm_mhz=None, hbm_peak=6557.4):
    """C3: SHA256d+Blake2B and Blake256+Ethash nonce search, nonce ranges sharded over ranks
    (rank r owns [r * count, (r + 1) * count)), one reduction per pair (hit count sum, winning
    nonce min); C4: Upsample (tunable) + Blake256 (fixed 512) over d0 in {640..1024} x
    register caps {none, r0, 32, 40, 48, 64, 96}. Fused vs unfused under the flushed-L2 protocol."""
    from paper_2007_01277_b200 import crypto as CR
    from paper_2007_01277_b200 import pairs as P
    grid = args.grid
    cgrids = sorted({grid, 2 * grid})  # every variant at its best of 1 and 2 waves of 148 x 2 blocks
    srcs = {k: open(os.path.join(P.KERNELS, "b200", k + ".mk")).read() for k in CR.MEMBERS}
    out = {"c3": [], "c4": None}
    for a, b in (("sha256d", "blake2b"), ("blake256", "ethash")):
        gmax = max(cgrids)  # per-block minimum arrays sized for the largest grid
        wa = CR.workload(a, CRYPTO_COUNTS[a], gmax, nonce0=rank * CRYPTO_COUNTS[a], target=1 << 12)
        wb = CR.workload(b, CRYPTO_COUNTS[b], gmax, nonce0=rank * CRYPTO_COUNTS[b], target=1 << 12,
                         npages=ETHASH_PAGES)
        img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload(stream)
        ka = hf.Module.kernel(srcs[a], grid=grid, specialize=img)
        kb = hf.Module.kernel(srcs[b], grid=grid, specialize=img)
        member_grid = {}
        for name, k in ((a, ka), (b, kb)):
            ts = {g: hf.time("single", k, None, img, g, warmup=2, reps=5, stream=stream)["iqm_us"] for g in cgrids}
            member_grid[name] = min(ts, key=ts.get)
        ga, gb = member_grid[a], member_grid[b]
        # fixed + fixed: one partition (fixed_partition_fuse); fixed + tunable (Blake256 +
        # Ethash): the tunable side gets d0 - 512 for each d0 tried
        # every point also tries per-interval register budgets (setmaxnreg): the fused kernel
        # no longer forces one register count on a 32-register hash and a 128-register Ethash
        best_r, traces = None, []
        for g in cgrids:
            for d0 in ((1024,) if b != "ethash" else (768, 896, 1024)):
                try:
                    r = hf.search(srcs[a], srcs[b], img, d0=d0, grid=g, reps=5, warmup=2, specialize=True,
                                  extra_caps=(64, 96, 128) if b == "ethash" else (), interval_regs=True)
                except hf.HFuseError:
                    continue
                traces += [(g, x["d1"], x["d2"], x["reg_cap"], round(x["us"], 1)) for x in r["trace"]]
                if best_r is None or r["best_time"] < best_r[0]["best_time"]:
                    best_r = (r, g)
        r, grid_f = best_r
        if r["interval_regs"]:
            m = hf.Module.fused_regs(srcs[a], srcs[b], r["d1"], r["d2"], *r["interval_regs"], grid=grid_f,
                                     specialize=img)
        else:
            m = hf.Module.fused(srcs[a], srcs[b], r["d1"], r["d2"], regcap=r["reg_cap"] or "off", grid=grid_f,
                                specialize=img)
        t = {mode: hf.time(mode, ka, kb, img, ga, gb, warmup=2, reps=10, stream=stream)["iqm_us"]
             for mode in ("sequential", "two_stream")}
        two_g = (ga, gb)
        for x in cgrids:  # the two-stream baseline at its best grid pair (as for the DL pairs)
            for y in cgrids:
                if (x, y) != (ga, gb):
                    tt = hf.time("two_stream", ka, kb, img, x, y, warmup=2, reps=10, stream=stream)["iqm_us"]
                    if tt < t["two_stream"]:
                        t["two_stream"], two_g = tt, (x, y)
        tf = hf.time("single", m, None, img, grid_f, warmup=2, reps=10, stream=stream)["iqm_us"]
        ta = hf.time("single", ka, None, img, ga, warmup=2, reps=10, stream=stream)["iqm_us"]
        tb = hf.time("single", kb, None, img, gb, warmup=2, reps=10, stream=stream)["iqm_us"]
        res = {"pair": f"{a}+{b}", "grid": grid_f, "grid_a": ga, "grid_b": gb, "two_stream_grids": list(two_g),
               "d1": r["d1"], "d2": r["d2"],
               "reg_cap": r["reg_cap"],
               "interval_regs": r["interval_regs"], "regs": m.info.regs,
               "blocks_per_sm": m.info.blocks_per_sm, "a_us": ta, "b_us": tb, "seq_us": t["sequential"],
               "two_stream_us": t["two_stream"], "fused_us": tf,
               "speedup": min(t["sequential"], t["two_stream"]) / tf,
               "nonces": {a: CRYPTO_COUNTS[a], b: CRYPTO_COUNTS[b]},
               "mhash_s_fused": (CRYPTO_COUNTS[a] + CRYPTO_COUNTS[b]) / tf,
               "search_trace": traces}
        if b == "ethash":
            res["dag_bytes"] = wb.dag_bytes
            res["dag_gbs_fused"] = CRYPTO_COUNTS[b] * 64 * 128 / (tf * 1e3)
        res["roofline"] = crypto_roofline({a: CRYPTO_COUNTS[a], b: CRYPTO_COUNTS[b]}, tf, sm_mhz, hbm_peak)
        # the single exchange: total hits + winning nonce over all ranks
        img_out = hf.Image(wa.image).merge(hf.Image(wb.image)).upload(stream)
        m.run(img_out, grid_f, stream)
        img_out.download(stream)
        hits = torch.tensor([int(img_out.array(f"{CR.MEMBERS[k]}_cnt")[0]) for k in (a, b)], dtype=torch.int64)
        win = torch.tensor([int(img_out.array(f"{CR.MEMBERS[k]}_bmin")[:grid_f].min()) for k in (a, b)],
                           dtype=torch.int64)
        if world > 1:
            import torch.distributed as dist
            hits, win = hits.cuda(), win.cuda()
            all_reduce(hits)
            all_reduce(win, "min")
        res["hits"] = hits.tolist()
        res["winning_nonce"] = win.tolist()
        out["c3"].append(res)
        del img, img_out
    # C4: Upsample + Blake256. Every variant at its best launch grid from the DL grid set:
    # each member alone (sequential), every grid pair (two-stream), every grid for the fused
    # kernel's search
    c4_grids = [296, 592, 1184, 2368]
    wu = P.MEMBERS["upsample"].sizes["full"](rank)
    wb = CR.workload("blake256", 1 << 21, max(c4_grids), nonce0=0, target=1 << 12)
    img = hf.Image(wu.image).merge(hf.Image(wb.image)).upload(stream)
    su = P.source("b200", "upsample")
    ku = hf.Module.kernel(su, grid=grid, specialize=img)
    kb = hf.Module.kernel(srcs["blake256"], grid=grid, specialize=img)
    alone = {}
    for name, k in (("upsample", ku), ("blake256", kb)):
        ts = {g: hf.time("single", k, None, img, g, warmup=2, reps=10, stream=stream)["iqm_us"] for g in c4_grids}
        alone[name] = min(ts, key=ts.get)
    gu, gbk = alone["upsample"], alone["blake256"]
    seq = hf.time("sequential", ku, kb, img, gu, gbk, warmup=2, reps=10, stream=stream)["iqm_us"]
    two, two_g = None, None
    for x in c4_grids:
        for y in c4_grids:
            tt = hf.time("two_stream", ku, kb, img, x, y, warmup=2, reps=10, stream=stream)["iqm_us"]
            if two is None or tt < two:
                two, two_g = tt, [x, y]
    sweep = []
    for g in c4_grids:
        for d0 in (640, 768, 896, 1024):
            try:
                r = hf.search(su, srcs["blake256"], img, d0=d0, grid=g, reps=5, warmup=2, specialize=True,
                              extra_caps=(32, 40, 48, 64, 96), interval_regs=True)
            except hf.HFuseError:
                continue
            for row in r["trace"]:
                sweep.append({"grid": g, "d0": d0, "d1": row["d1"], "reg_cap": row["reg_cap"],
                              "interval_regs": row.get("interval_regs"), "us": round(row["us"], 2),
                              "occupancy": round(row["occupancy"], 3)})
    best = min(sweep, key=lambda x: x["us"])
    out["c4"] = {"pair": "upsample+blake256", "seq_us": seq, "two_stream_us": two, "grid_a": gu, "grid_b": gbk,
                 "two_stream_grids": two_g, "best": best,
                 "speedup": min(seq, two) / best["us"], "sweep": sweep}
    # C4 pair roofline: max(Upsample's HBM time, BLAKE-256's issue time)
    rb = crypto_roofline({"blake256": 1 << 21}, best["us"], sm_mhz, hbm_peak)
    if rb is not None:
        t_hbm = wu.bytes / (hbm_peak * 1e3)
        t_roof = max(t_hbm, rb["issue_us"])
        out["c4"]["roofline"] = {"bound": "hbm" if t_hbm >= rb["issue_us"] else "issue", "roofline_us": t_roof,
                                 "frac": t_roof / best["us"], "hbm_us": t_hbm, "issue_us": rb["issue_us"],
                                 "alu_pipe_us": rb["alu_pipe_us"]}
    return out



def stream_ceilings(hf, P, results, work, grids, flush, stream):
    """Mix-matched HBM ceiling of every pair: plain 128-bit streaming kernels
    (kernels/probe/stream*.mk, one or four loads in flight per thread) reading and writing the
    pair's algorithmic read / write bytes, best over both forms and the fused grids, timed under
    the same protocol as the pairs. Adds ceiling_us / ceiling_frac (= ceiling / fused) to each
    result: how close the fused kernel is to what HBM delivers for that read:write mix and
    size, where the copy roofline assumes one fixed mix."""
    forms = {k: open(os.path.join(P.KERNELS, "probe", k + ".mk")).read() for k in ("stream", "stream4")}
    for res in results:
        a, b = res["pair"].split("+")
        r, w = work[a].read + work[b].read, work[a].write + work[b].write
        img = hf.Image(f"array s_src float32 {r // 4} zero\narray s_dst float32 {max(w, 64) // 4} zero\n"
                       f"scalar s_nr4 int32 {r // 16}\nscalar s_nw4 int32 {w // 16}\n").upload(stream)
        best = None
        for name, text in forms.items():
            m = hf.Module.kernel(text, grid=grids[0], specialize=img)
            for g in sorted(set(grids) | {2 * x for x in grids}):
                t = hf.time("single", m, None, img, g, warmup=3, reps=30, flush_l2=flush, stream=stream)["iqm_us"]
                if best is None or t < best[0]:
                    best = (t, name, g)
            del m
        res["ceiling_us"] = best[0]
        res["ceiling_kernel"] = f"{best[1]}@{best[2]}"
        res["ceiling_frac"] = best[0] / res["fused_us"]
        del img


def best_two_stream(hf, ka, kb, img, ga, gb, grids, flush, stream):
    """The two-stream baseline with the same grid freedom as the fused kernel: timed at the
    members' best grids alone, every other (grid_a, grid_b) pair screened with 15 repetitions
    and the best re-timed like the rest (concurrent kernels share the SMs, so the members' best
    grids alone need not be the pair's best; profiles/r01_probe_two_stream_grids.json).
    Returns (timing dict, grid_a, grid_b)."""
    two = hf.time("two_stream", ka, kb, img, ga, gb, warmup=5, reps=60, flush_l2=flush, stream=stream)
    screen = {(x, y): hf.time("two_stream", ka, kb, img, x, y, warmup=2, reps=15, flush_l2=flush,
                              stream=stream)["iqm_us"]
              for x in grids for y in grids if (x, y) != (ga, gb)}
    if screen:
        bx, by = min(screen, key=screen.get)
        if screen[(bx, by)] < two["iqm_us"]:
            alt = hf.time("two_stream", ka, kb, img, bx, by, warmup=5, reps=60, flush_l2=flush, stream=stream)
            if alt["iqm_us"] < two["iqm_us"]:
                return alt, bx, by
    return two, ga, gb


def ratio_study(hf, P, pair_list, src, shape, rank, grids, d0s, flush, stream, member_us, args):
    """The paper's workload-ratio experiment: every pair with
    its second member's batch rescaled so the unfused times stand at t_b / t_a = r for each r in
    --ratios, each point fused, searched exhaustively and compared like the main table (the
    model pre-filter, K = 3, missed BN + Upsample at r = 2 by 13 %). Outside the timed step."""
    ratios = [float(x) for x in args.ratios.split(",")]
    rows = []
    for a, b in pair_list:
        for r in ratios:
            wa = P.MEMBERS[a].sizes[shape](rank)
            f = r * member_us[a] / member_us[b]
            for attempt in range(2):
                # batch scale from the natural-size times, then one correction from the
                # measured ratio (a launch's fixed cost makes time not quite linear in batch)
                wb, nb = P.scaled(b, f, shape, seed=rank)
                img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload(stream)
                ka = hf.Module.kernel(src[a], grid=grids[0], specialize=img)
                kb = hf.Module.kernel(src[b], grid=grids[0], specialize=img)
                alone = {}
                for name, k in ((a, ka), (b, kb)):
                    ts = {g: hf.time("single", k, None, img, g, warmup=2, reps=10, flush_l2=flush,
                                     stream=stream)["iqm_us"] for g in grids}
                    g = min(ts, key=ts.get)
                    alone[name] = (g, ts[g])
                got = alone[b][1] / alone[a][1]
                if attempt == 1 or abs(got / r - 1.0) <= 0.05:
                    break
                f_next = f * r / got
                if P.scaled(b, f_next, shape)[1] == nb:
                    break
                f = f_next
                del ka, kb, img
            best, grid = None, None
            for d0 in d0s:
                for g in grids if d0 == 1024 else [2 * x for x in grids]:
                    rg = hf.search(src[a], src[b], img, d0=d0, grid=g, reps=args.search_reps, warmup=2,
                                   specialize=True, flush_l2=flush, granularity=args.granularity)
                    if best is None or rg["best_time"] < best["best_time"]:
                        best, grid = rg, g
            cap = best["reg_cap"]
            m = hf.Module.fused(src[a], src[b], best["d1"], best["d2"], regcap=cap if cap else "off", grid=grid,
                                specialize=img)
            tf = hf.time("single", m, None, img, grid, warmup=5, reps=60, flush_l2=flush, stream=stream)["iqm_us"]
            (ga, ta), (gb, tb) = alone[a], alone[b]
            seq = hf.time("sequential", ka, kb, img, ga, gb, warmup=5, reps=60, flush_l2=flush, stream=stream)["iqm_us"]
            two, tga, tgb = best_two_stream(hf, ka, kb, img, ga, gb, grids, flush, stream)
            rows.append({"pair": f"{a}+{b}", "target_ratio": r, "ratio": round(tb / ta, 3), "batch_b": nb,
                         "a_us": round(ta, 2), "b_us": round(tb, 2), "grid": grid, "d0": best["d1"] + best["d2"],
                         "d1": best["d1"], "d2": best["d2"], "reg_cap": cap, "fused_us": round(tf, 2),
                         "seq_us": round(seq, 2), "two_stream_us": round(two["iqm_us"], 2),
                         "two_stream_grids": [tga, tgb], "speedup": round(min(seq, two["iqm_us"]) / tf, 4)})
            del m, ka, kb, img
    geo = {}
    for r in ratios:
        sp = [x["speedup"] for x in rows if x["target_ratio"] == r]
        geo[str(r)] = math.exp(sum(math.log(v) for v in sp) / len(sp)) if sp else None
    return {"how": "second member's batch scaled to t_b/t_a = r (members timed alone at their best grids); "
                   "fused search over d0 x grids x splits x caps (exhaustive); "
                   "two-stream at its best grid pair", "rows": rows, "speedup_geomean": geo}


def e2e_step(hf, torch, P, pair_list, fused, work, keys, pgrid, stream, args):
    """Host-buffer end-to-end step through hf_launch (the C-ABI call): every input tensor of the
    step (an array no kernel writes) goes pinned host -> HBM once, the ten fused kernels run,
    and each pair's outputs (every array it writes) come back HBM -> pinned host. Arrays a kernel
    writes but never reads (hf_module_param_reads: no loads, no atomics) are not uploaded; a
    written array that is also read (histogram bins) is uploaded per pair from its host zeros.
    Pipelined over three streams (upload / fused kernels / download; PCIe is full duplex): a
    pair waits only for its own inputs, outputs drain while later pairs run. Outputs use per-pair
    device buffers; cross-step reuse of any buffer waits on the events of its last user."""
    host, scal = {}, {}
    for k in keys:
        arrays, scalars = _image_arrays(hf, work[k].image)
        scal.update(scalars)
        for name, (dtype, n, init) in arrays.items():
            h = torch.empty(n, dtype=dtype, pin_memory=True)
            if init is not None:
                h.copy_(torch.from_numpy(init))
            else:
                h.zero_()
            host[name] = h
    written = {p["name"] for a, b in pair_list for p in fused[(a, b)].params if p["array"] and p["written"]}
    shared = {}  # input tensors: one device copy per step, shared by the pairs that read them
    plan = []    # per pair: (module, grid, shared inputs, per-pair uploads, downloads, launch args)
    last_reader = {}
    for i, (a, b) in enumerate(pair_list):
        m = fused[(a, b)]
        ins, ups, downs, args_ = [], [], [], {}
        for p in m.params:
            if not p["array"]:
                args_[p["name"]] = scal[p["name"]]
                continue
            h = host[p["name"]]
            if p["name"] not in written:
                if p["name"] not in shared:
                    shared[p["name"]] = torch.empty(h.numel(), dtype=h.dtype, device="cuda")
                args_[p["name"]] = shared[p["name"]]
                ins.append(p["name"])
                last_reader[p["name"]] = i
                continue
            d = torch.empty(h.numel(), dtype=h.dtype, device="cuda")
            args_[p["name"]] = d
            if p["read"]:
                ups.append((d, h))
            downs.append((h, d))
        plan.append((m, pgrid[(a, b)], ins, ups, downs, args_))
    # downloads alternate over HF_E2E_DOWN_STREAMS streams (default 1; probe: more copy engines)
    n_down = max(1, int(os.environ.get("HF_E2E_DOWN_STREAMS", "1")))
    s_up, s_downs = torch.cuda.Stream(), [torch.cuda.Stream() for _ in range(n_down)]
    n = len(plan)
    ev_in = {name: torch.cuda.Event() for name in shared}
    ev_up = [torch.cuda.Event() for _ in range(n)]
    ev_k = [torch.cuda.Event() for _ in range(n)]
    ev_dn = [torch.cuda.Event() for _ in range(n)]

    def one_step(first):
        sent = set()
        for i, (m, g, ins, ups, downs, args_) in enumerate(plan):
            with torch.cuda.stream(s_up):
                for name in ins:
                    if name in sent:
                        continue
                    if not first:
                        s_up.wait_event(ev_k[last_reader[name]])  # last step's readers are done
                    shared[name].copy_(host[name], non_blocking=True)
                    ev_in[name].record(s_up)
                    sent.add(name)
                if not first:
                    s_up.wait_event(ev_k[i])
                for d, h in ups:
                    d.copy_(h, non_blocking=True)
                ev_up[i].record(s_up)
            for name in ins:
                stream.wait_event(ev_in[name])
            stream.wait_event(ev_up[i])
            if not first:
                stream.wait_event(ev_dn[i])       # its outputs of the previous step are downloaded
            m.launch(args_, grid=g, stream=stream)
            ev_k[i].record(stream)
            s_down = s_downs[i % n_down]
            with torch.cuda.stream(s_down):
                s_down.wait_event(ev_k[i])
                for h, d in downs:
                    h.copy_(d, non_blocking=True)
                ev_dn[i].record(s_down)
    h2d = sum(host[name].numel() * host[name].element_size() for name in shared) + \
        sum(h.numel() * h.element_size() for _, _, _, ups, _, _ in plan for _, h in ups)
    d2h = sum(h.numel() * h.element_size() for _, _, _, _, downs, _ in plan for h, _ in downs)
    one_step(True)
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 5))
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    s_up.wait_event(s0)
    for s_down in s_downs:
        s_down.wait_event(s0)
    for i in range(steps):
        one_step(False)
    for s_down in s_downs:
        stream.wait_stream(s_down)
    s1.record(stream)
    torch.cuda.synchronize()
    us = s0.elapsed_time(s1) * 1000.0 / steps
    return {"value": us, "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": steps,
            "pipeline": "3 streams (upload / fused kernels / download); each input tensor uploaded once "
                        "per step; per-pair outputs downloaded; pure outputs not uploaded"}


def _image_arrays(hf, text):
    """Host initial contents of an image's arrays, generated by libhfuse's host-side
    memimage implementation (the same splitmix64 stream the device fill produces)."""
    import torch
    img = hf.Image(text).materialize()
    arrays, scalars = {}, {}
    for line in text.splitlines():
        f = line.split()
        if not f:
            continue
        if f[0] == "scalar":
            scalars[f[1]] = int(f[3]) if f[2] == "int32" else float(f[3])
            continue
        name, typ, n = f[1], f[2], int(f[3])
        dtype = torch.int32 if typ == "int32" else torch.float32
        arrays[name] = (dtype, n, img.array(name))
    return arrays, scalars


if __name__ == "__main__":
    sys.exit(main())
