#!/usr/bin/env python
"""Benchmark of the chaotic-iteration PRNG hot path (arXiv 1112.5239) on B200.

Metric (BASELINE.json): 32-bit random numbers/s, whole job, and the fraction
of the HBM write roofline.  One step = one prng_generate call of BASELINE
configs[1] per GPU: V1 (Alg. 4, xor128 + neighbour combination), 2^20 streams
x 128 numbers, stored to HBM (512 MiB per step).  L2 is flushed between
timed calls so the 24 MiB of state start each call in HBM, and each call is
CHARGED the write-back of the output lines it left dirty in L2: a step's time
is call + the following flush, minus the flush alone.
Multi-GPU (one process per GPU): every rank owns 2^20 consecutive streams of
one global stream space (weak scaling); the store path has no collective at
all.  `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N processes.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, plain single-threaded C) on
this host on the same C2 workload (every step a full 2^20 x 128 call): the
paper ships no code, so the oracle is the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "32-bit random numbers/sec at 1/2/4/8 B200; % of HBM write roofline"
UNIT = "numbers/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
CFG = W.CONFIGS["C2"]
S_PER_GPU, N_PER_STREAM = CFG["n_streams"], CFG["n"]
STATE_BYTES_V1 = 24  # per stream, read once + written once per call


def env_rank():
    r = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    lr = int(os.environ.get("LOCAL_RANK", str(r)))
    return r, ws, lr


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)", d
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


def write_only_peak():
    """Write-only HBM bandwidth measured on this pool's B200 by
    tools/pattern_bench.py (torch fill of 512 MiB, profiles/r1_hbm_write_patterns.json)."""
    p = os.path.join(ROOT, "profiles", "r1_hbm_write_patterns.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh).get("torch_fill_512MiB", 0.0)) or None
    return None


def ncu_traffic():
    """dram bytes per launch of the V1 store kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_v1_store.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch")
    return None


# Issue peak (one warp instruction per scheduler per clock = 148 SMs x 4 x 32
# lanes x 1.965 GHz) -- reported beside the pipe roofline of the
# compute-bound rows, not as it.
N_SM = 148
SM_MAX_HZ = 1.965e9
ISSUE_PEAK_TLANE = N_SM * 4 * 32 * SM_MAX_HZ / 1e12
# ncu capture kind (tools/prof_kernels.py) -> (secondary key, numbers per launch)
NCU_KINDS = {"v2": ("c3_v2_store", 2**20 * 64), "v0": ("v0_store", 2**20 * 128), "v3": ("v3_store", 2**20 * 128),
             "v4": ("v4_store", 2**20 * 128), "consume": ("c5_v1_consume", 2**20 * 1024),
             "consume_v0": ("c5_v0_consume", 2**20 * 1024), "consume_v2": ("c5_v2_consume", 2**20 * 1024),
             "consume_v3": ("c5_v3_consume", 2**20 * 1024), "battery": ("v1_battery", 2**20 * 1024),
             "cbg": ("cbg_encrypt", 2**18 * 1024)}


def ncu_captures():
    """The newest committed ncu capture of each secondary kernel
    (profiles/r*_ncu_summary.json, written by tools/ncu_summary.py from
    `ncu --set full` reports): {secondary key: (capture, numbers per launch,
    source file)}."""
    import glob

    # newest by name (r1a < ... < r1zc < r2a): mtimes of a fresh checkout carry no order
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    out = {}
    for f in reversed(files):
        with open(f) as fh:
            caps = json.load(fh).get("captures", {})
        for kind, (key, numbers) in NCU_KINDS.items():
            if key in out:
                continue
            for c in caps.get(kind, []):
                if c.get("warp_insts") and c.get("duration") and c.get("sm_clock"):
                    out[key] = (c, numbers, os.path.relpath(f, ROOT))
                    break
    return out


def pipe_roofline(rate: float, cap: dict, numbers: int, src: str) -> dict:
    """Roofline of a compute-bound row against its BINDING integer pipe.

    ncu gives, for one launch of `numbers` numbers, the busy fraction of the
    ALU and heavy-FMA pipes (sm__pipe_{alu,fmaheavy}_cycles_active, % of peak
    sustained over the elapsed cycles) and of the L1/shared-memory data pipe
    (l1tex__data_pipe_lsu_wavefronts: the consumers' histogram atomics); the
    busiest of the three is the binding one.  Busy pipe-cycles per number =
    fraction x duration x SM clock x 148 SMs / numbers; `achieved` = that x
    the live bench rate, `peak` = 148 SMs x the max SM clock (the pipe busy
    every cycle on every SM), so `frac` is the live rate's busy fraction of
    the binding pipe.  The issue-slot figure (instructions per number x rate
    over the 4-scheduler issue peak) is reported beside it."""
    alu = cap.get("pipe_alu_cycles_pct", 0.0) / 100.0
    heavy = cap.get("pipe_fmaheavy_cycles_pct", 0.0) / 100.0
    # the L1/shared data pipe (one wavefront per SM per cycle): the consumers'
    # bank-conflicted histogram atomics load it as much as the ALU
    lsu = cap.get("lsu_data_pct", 0.0) / 100.0
    pipe, busy = max((("alu", alu), ("fmaheavy", heavy), ("lsu_data", lsu)), key=lambda kv: kv[1])
    cyc_per_number = busy * cap["duration"] * cap["sm_clock"] * N_SM / numbers
    peak = N_SM * SM_MAX_HZ
    ach = rate * cyc_per_number
    ipn = cap["warp_insts"] * 32 / numbers
    return {"bound": pipe, "achieved": ach / 1e12, "peak": peak / 1e12, "unit": "T pipe-cycles/s",
            "frac": ach / peak, "pipe_cycles_per_number": cyc_per_number,
            "ncu_busy_frac": {"alu": alu, "fmaheavy": heavy, "lsu_data": lsu}, "kernel": cap.get("kernel"),
            "source": f"{src} (ncu --set full: sm__pipe_*_cycles_active, l1tex__data_pipe_lsu_wavefronts, "
                      "gpu__time_duration, "
                      "sm__cycles_elapsed.avg.per_second); peak = 148 SMs x 1.965 GHz",
            "issue": {"inst_per_number": ipn, "achieved": rate * ipn / 1e12, "peak": ISSUE_PEAK_TLANE,
                      "unit": "T lane-inst/s", "frac": rate * ipn / 1e12 / ISSUE_PEAK_TLANE}}


class ClockSampler:
    """NVML clock / throttle-reason sampling during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


def cpu_model() -> str | None:
    """Host CPU model (/proc/cpuinfo), reported beside every CPU timing."""
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or None


def time_oracle(seconds: float = 10.0, max_calls: int = 64):
    """The oracle as it stands, single thread, on the C2 workload (full 2^20
    streams x 128 per call), as many calls as fit in ~`seconds`."""
    import oracle as O

    st = O.init_states(W.V1, W.SEEDS[0], 0, S_PER_GPU)
    calls, t0 = 0, time.perf_counter()
    while True:
        O.generate(W.V1, st, N_PER_STREAM)
        calls += 1
        el = time.perf_counter() - t0
        if el >= seconds or calls >= max_calls:
            break
    numbers = calls * S_PER_GPU * N_PER_STREAM
    return {
        "value": numbers / el,
        "unit": UNIT,
        "cores": 1,
        "cpu_model": cpu_model(),
        "kind": "oracle",
        "sample": f"{calls} call(s) of the full C2 workload (V1, 2^20 streams x 128) = {numbers} numbers, "
                  f"single-threaded C oracle, {el:.1f} s wall",
    }


def _oracle_slice(job):
    """One process of the all-cores baseline: `calls` C2 calls over streams
    [first, first + count) with the unmodified oracle."""
    first, count, calls = job
    import oracle as O

    st = O.init_states(W.V1, W.SEEDS[0], first, count)
    t0 = time.perf_counter()
    for _ in range(calls):
        O.generate(W.V1, st, N_PER_STREAM)
    return time.perf_counter() - t0


def time_oracle_all_cores(calls: int = 16):
    """The same oracle in P = nproc processes over disjoint 32-stream groups of
    the full C2 stream space (one process per core; nothing in the oracle is
    changed), `calls` calls of the full workload; time = the slowest worker's
    generate loop (process start-up excluded)."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    P = max(1, os.cpu_count() or 1)
    groups = S_PER_GPU // 32
    jobs = [((groups * r // P) * 32, (groups * (r + 1) // P - groups * r // P) * 32, calls) for r in range(P)]
    t0 = time.perf_counter()
    # a crashed worker raises BrokenProcessPool (a Pool would respawn forever)
    with ProcessPoolExecutor(P, mp_context=mp.get_context("spawn")) as ex:
        worker_s = list(ex.map(_oracle_slice, jobs, timeout=300))
    wall = time.perf_counter() - t0
    el = max(worker_s)
    numbers = calls * S_PER_GPU * N_PER_STREAM
    return {"value": numbers / el, "unit": UNIT, "cores": P, "cpu_model": cpu_model(), "kind": "oracle",
            "sample": f"{calls} call(s) of the full C2 workload split over {P} processes (one per core) by "
                      f"32-stream groups; slowest worker {el:.1f} s ({wall:.1f} s wall incl. process start)"}


# --------------------------------------------------------------------------
def run_reference(args):
    """The reference arm: the oracle as it stands, single-threaded on this
    host's cores, on the SAME workload as our arm -- every step one full C2
    call (V1, 2^20 streams x 128 numbers, state carried across steps).  Under
    torchrun only rank 0 runs; the others exit 0 without work."""
    rank, ws, _ = env_rank()
    if rank != 0:
        return 0
    import oracle as O

    S, n = S_PER_GPU, N_PER_STREAM
    st = O.init_states(W.V1, W.SEEDS[0], 0, S)
    # one untimed full call calibrates the per-step cost; if K + W full calls
    # would exceed the budget, every step is a bounded sample: the first S'
    # streams (whole 32-stream groups) of the same workload
    t0 = time.perf_counter()
    O.generate(W.V1, st, n)
    t_call = time.perf_counter() - t0
    budget_s = 150.0
    if (args.steps + args.warmup) * t_call > budget_s:
        S = max(32, int(S * budget_s / ((args.steps + args.warmup) * t_call)) // 32 * 32)
        st = O.init_states(W.V1, W.SEEDS[0], 0, S)
    for _ in range(args.warmup):
        O.generate(W.V1, st, n)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.generate(W.V1, st, n)
    el = time.perf_counter() - t0
    v = args.steps * S * n / el
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v,
        "unit": UNIT,
        "n_gpus": ws if ws > 1 else max(1, args.gpus),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded; SplitMix64 per-stream seeding, seed 0x0123456789ABCDEF)",
        "config": {"workload": "C2 (BASELINE configs[1]): V1 Alg.4 xor128 + neighbour combination (default C=32 "
                               f"arrays), {S} streams x {n} numbers per step", "variant": "v1",
                   "streams_per_gpu": S_PER_GPU, "n_per_stream": n, "same_config_as_ours": True,
                   "streams_per_step_timed": S},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": (f"{args.steps} steps x the full C2 call ({S} streams x {n} numbers)"
                                    if S == S_PER_GPU else
                                    f"{args.steps} steps x the first {S} of the C2 call's {S_PER_GPU} streams x {n} "
                                    f"numbers (bounded: K + W full calls would take "
                                    f"{(args.steps + args.warmup) * t_call:.0f} s)")
                                   + ", single-threaded C oracle, rank 0 only"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class L2Flush:
    """Untimed L2 flush between timed calls: a 256 MiB write (> the 126 MB
    L2) followed by a 256 MiB read.  The write alone leaves up to ~126 MB of
    the flush buffer's own DIRTY lines in L2, whose write-back to HBM would
    then land inside the next timed call (measured: write-only flush 1.484e12
    vs write+read 1.51-1.53e12 numbers/s, tools/exp_flush.py,
    profiles/experiments/s32_flush*.json); the read pass (an int32 amax:
    a pure read reduction, no dtype-cast copy) writes them back
    before the timer starts and leaves L2 full of clean, unrelated lines, so
    the timed call still finds its state planes in HBM."""

    def __init__(self, torch, dev):
        self.w = torch.empty(64 * 2**20, dtype=torch.int32, device=dev)
        self.r = torch.ones(64 * 2**20, dtype=torch.int32, device=dev)
        self.acc = torch.empty((), dtype=torch.int32, device=dev)
        self.torch = torch

    def __call__(self, k: int) -> None:
        self.w.fill_(k)
        self.acc.copy_(self.torch.amax(self.r))


def run_ours(args):
    import torch

    import paper_1112_5239_b200 as P

    rank, ws, lr = env_rank()
    # one process per GPU; CIPRNG_BENCH_BACKEND=gloo lets tests drive the
    # multi-rank path with several ranks on one GPU (device = local rank mod #GPUs)
    lr = lr % max(1, torch.cuda.device_count())
    if ws > 1:
        import torch.distributed as dist

        torch.cuda.set_device(lr)
        backend = os.environ.get("CIPRNG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(lr)
        dist = None
    dev = torch.device("cuda", lr)
    S, n = args.streams or S_PER_GPU, args.rounds or N_PER_STREAM
    g = P.ChaoticPRNG(W.SEEDS[0], S * ws, P.V1, shard=(rank * S, S), store_path=args.store_path)
    out = torch.empty((S, n), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        g.generate(n, out=out)
    launches_per_step = g.info().kernel_launches
    store_path_used = g.info().store_path
    torch.cuda.synchronize()

    # (1) headline: L2 flushed between timed steps (L2Flush: 256 MiB write +
    # read > the 126 MB L2, so the 24 MiB of state planes start every call in
    # HBM), each step timed with CUDA events on the launching stream.  A call
    # ends with up to ~13 % of its output still dirty in L2; the flush after
    # it pays that write-back.  So a step is timed as [call + the following
    # flush] and CHARGED that span minus the mean time of a flush that
    # follows a flush (clean L2): every byte the call writes reaches HBM
    # inside its charged time.  The flush after step k is the pre-flush of
    # step k+1.
    flush = L2Flush(torch, dev)
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(lr) as clk:
        # the W warm-up steps again, flush included, right before the timed
        # region: after any idle gap (NVML start-up, the flush buffer's
        # allocation) the first call runs ~2x slow (profiles/experiments/
        # s48_step_times.json: 178 vs 87 us), which would bias a short --steps
        for k in range(args.warmup):
            flush(k)
            g.generate(n, out=out)
        flush(0)
        barrier()
        torch.cuda.synchronize()
        for k in range(args.steps):
            ev[k][0].record(stream)
            g.generate(n, out=out)
            ev[k][1].record(stream)
            flush(k + 1)
            ev[k][2].record(stream)
        # the flush alone, after a flush (nothing of ours dirty in L2)
        for k in range(args.steps):
            flush(k)
            fev[k][0].record(stream)
            flush(k + 1)
            fev[k][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    event_ms = sum(a.elapsed_time(b) for a, b, _ in ev)
    flush_alone_ms = sum(a.elapsed_time(b) for a, b in fev) / args.steps
    charged_ms = sum(a.elapsed_time(c) for a, _, c in ev) - args.steps * flush_alone_ms
    # never credit the call with a flush faster than the one that followed it
    charged_ms = max(charged_ms, event_ms)
    t = torch.tensor([charged_ms, event_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, event_ms = float(t[0].item()), float(t[1].item())
    numbers = args.steps * S * n * ws
    value = numbers / (total_ms / 1e3)
    del flush

    # (2) steady state: back-to-back calls with no flush (no per-launch events:
    # they would break the programmatic-dependent-launch overlap).  The output
    # is stored L2-evict-first, so across calls the state planes stay
    # L2-resident -- the regime of a generator serving calls continuously.
    for _ in range(args.warmup):  # hot GPU at the first timed call (s48)
        g.generate(n, out=out)
    barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for k in range(args.steps):
        g.generate(n, out=out)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    steady_ms = t_start.elapsed_time(t_end)
    t = torch.tensor([steady_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    steady_ms = float(t.item())
    steady_value = numbers / (steady_ms / 1e3)

    # (3) the same steady state replayed from a CUDA graph of 10 calls (single
    # process only: a capture must not race the NCCL watchdog thread)
    graph_value = None
    try:
        if ws > 1:
            raise RuntimeError("skipped under torch.distributed")
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs, capture_error_mode="thread_local"):
            for _ in range(10):
                g.generate(n, out=out)
        reps = max(1, args.steps // 10)
        graph.replay()
        torch.cuda.synchronize()
        barrier()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        for _ in range(reps):
            graph.replay()
        b_ev.record(stream)
        torch.cuda.synchronize()
        graph_value = reps * 10 * S * n / (a_ev.elapsed_time(b_ev) / 1e3)
        del graph
    except Exception as e:  # never lose the headline over the graph variant
        graph_value = {"error": repr(e)[:200]}

    # ---- end-to-end through the public API with a pinned host buffer
    host = torch.empty((S, n), dtype=torch.int32, pin_memory=True)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    g.generate_host(n, out=host)  # warm (staging buffers, copy stream)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        g.generate_host(n, out=host)
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    e2e_value = e2e_steps * S * n * ws / e2e_s
    # the bound of the e2e path: a plain pinned device->host copy of the same
    # bytes (torch, no generation) on this GPU's PCIe link
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host.copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    d2h_gbs = e2e_steps * 4 * S * n / (time.perf_counter() - t0) / 1e9

    # ---- roofline of the dominant (only) kernel: SURVEY s8(d) counts 4 B
    # written per number; the state (24 B read + 24 B written per stream per
    # call) is reported beside it, not in `achieved`
    peak, peak_src, peaks = measured_peaks()
    out_bytes = 4 * S * n
    state_bytes = 2 * STATE_BYTES_V1 * S
    avg_kern_s = total_ms / args.steps / 1e3       # charged time per launch (one launch per step)
    achieved = out_bytes / avg_kern_s / 1e9
    traffic = ncu_traffic()

    secondary = {}
    if not args.no_secondary:
        secondary = measure_secondary(P, torch, dev, args)
        for key, (cap, numbers_launch, src) in ncu_captures().items():
            if key in secondary:
                secondary[key]["roofline"] = pipe_roofline(secondary[key]["value"], cap, numbers_launch, src)

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic (seeded; SplitMix64 per-stream seeding, seed 0x0123456789ABCDEF)",
        "config": {
            "workload": ("C2 (BASELINE configs[1]): " if (S, n) == (S_PER_GPU, N_PER_STREAM) else "EXPERIMENT: ")
                        + "V1 Alg.4 xor128 + neighbour combination (default C=32 arrays), "
                        f"{S} streams x {n} numbers per GPU per step, stored to HBM",
            "variant": "v1",
            "streams_per_gpu": S,
            "n_per_stream": n,
            "global_streams": S * ws,
            "store_path": {1: "direct", 2: "tma"}.get(store_path_used, str(store_path_used)),
            "l2": "L2 flushed between timed steps (256 MiB write then 256 MiB read); each step charged its "
                  "deferred write-back (call + following flush - flush alone); output "
                  f"{4 * S * n >> 20} MiB per step per GPU, state {STATE_BYTES_V1 * S >> 20} MiB",
            "parallelism": f"stream-sharded x{ws} (no collective on the store path)",
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "kernel": "v1_fast_kernel<StoreSink>",
            "alg_bytes_per_launch": out_bytes,
            "alg_bytes_rule": "4 B written per number (SURVEY s8(d) C2); state reported separately",
            "state_bytes_per_launch": state_bytes,
            "achieved_incl_state": (out_bytes + state_bytes) / avg_kern_s / 1e9,
            "avg_kernel_ms": avg_kern_s * 1e3,
            "timing": "charged: per step (call + following L2 flush) - mean(flush after a flush); the call's "
                      "deferred write-back of dirty output lines is inside its time",
            "event_only_ms": event_ms / args.steps,
            "deferred_writeback_ms": (total_ms - event_ms) / args.steps,
            "flush_alone_ms": flush_alone_ms,
            "peak_source": peak_src,
            # the metric's "% of HBM write roofline" against a write-only stream
            # (a copy peak counts read + write turnarounds a writer does not pay)
            "write_only_peak": write_only_peak(),
            "frac_of_write_only_peak": (achieved / write_only_peak()) if write_only_peak() else None,
        },
        "e2e": {
            "value": e2e_value,
            "unit": UNIT,
            "h2d_bytes_per_step": 0,
            "d2h_bytes_per_step": 4 * S * n,
            "api": "prng_generate_host (pinned host buffer, chunked generate + D2H overlap)",
            "steps": e2e_steps,
            "d2h_copy_gbs": d2h_gbs,
            "frac_of_d2h_copy": e2e_value / ws * 4 / 1e9 / d2h_gbs,
            "bound": "PCIe device->host: the e2e rate over a plain pinned copy of the same bytes",
        },
        "steady_state": {
            "value": steady_value,
            "unit": UNIT,
            "ms_per_step": steady_ms / args.steps,
            "frac": out_bytes / (steady_ms / args.steps / 1e3) / 1e9 / peak,
            "note": "back-to-back calls, no L2 flush: output stored evict-first, so the 24 MiB of state "
                    "planes stay L2-resident across calls (only the output reaches HBM)",
            "cuda_graph_value": graph_value,
        },
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    if secondary:
        line["secondary"] = secondary
    # the paper's own figures, context only (other hardware, and
    # its ~20 GS/s were measured without storing the numbers)
    ctx = {"source": "PAPER.md P:1026-1057 via BASELINE.md; Tesla C1060 / GTX 280 (GT200, 240 cores)",
           "optimized_xor64_no_store_numbers_per_s": 2.0e10,
           "naive_listing1_no_store_numbers_per_s": 2.75e9,
           "bbs_numbers_per_s": 7.0e8,
           "headline_over_optimized_no_store": value / 2.0e10}
    if "c5_v1_consume" in secondary:
        ctx["consume_over_optimized_no_store"] = secondary["c5_v1_consume"]["value"] / 2.0e10
    if "c3_v2_store" in secondary:
        ctx["v2_store_over_bbs"] = secondary["c3_v2_store"]["value"] / 7.0e8
    for key, row, ref in (("v3_consume_over_optimized_no_store", "c5_v3_consume", 2.0e10),
                          ("v0_consume_over_naive_no_store", "c5_v0_consume", 2.75e9),
                          ("v2_consume_over_bbs", "c5_v2_consume", 7.0e8)):
        if row in secondary:
            ctx[key] = secondary[row]["value"] / ref
    line["paper_context"] = ctx
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = time_oracle(args.cpu_seconds)
        try:
            line["cpu_baseline_all_cores"] = time_oracle_all_cores()
        except Exception as e:  # never lose the headline over the extra baseline
            line["cpu_baseline_all_cores"] = {"error": repr(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    g.close()
    if dist:
        dist.destroy_process_group()
    return 0


def _c4_write_fracs(per_gpu: float) -> dict:
    """SURVEY s8(d) C4 "per-GPU % of write peak": 4 B written per number over
    the measured copy peak (MEASURED_PEAKS.json) and the write-only fill."""
    peak, _, _ = measured_peaks()
    wo = write_only_peak()
    gbs = per_gpu * 4 / 1e9
    out = {"per_gpu_write_gbs": gbs, "per_gpu_frac_of_copy_peak": gbs / peak}
    if wo:
        out["per_gpu_frac_of_write_only_peak"] = gbs / wo
    return out


def _hist_chi2(hist) -> dict:
    """SURVEY s8(d) C5 "chi^2_255 sane": Pearson chi^2 of the 256-bin top-byte
    histogram against uniform (host-side float on the final integer counts)
    and its upper-tail p-value (scipy's chi2 survival function)."""
    from scipy.stats import chi2

    h = [int(v) for v in hist]
    tot = sum(h)
    e = tot / 256.0
    x2 = sum((v - e) ** 2 for v in h) / e
    p = float(chi2.sf(x2, 255))
    return {"hist_chi2_255": x2, "hist_chi2_p": p, "hist_chi2_sane": 1e-6 < p < 1 - 1e-6}


def measure_c5_sharded(P, torch, dev, timed, calls: int = 10):
    """C5 (BASELINE configs[4]) as a job over every rank: V1 consumer mode on
    a global stream space of 2^20 streams per GPU (rank r owns the contiguous
    range [r 2^20, (r+1) 2^20)), n = 1024 per call; each call is the fused
    consume kernel followed by ONE all-reduce (NCCL under torchrun, SUM) of
    the 258 u64 statistics -- the a7 row, the path's only collective.  Timed
    per call with CUDA events around consume + all-reduce (L2 flushed before
    each call), max over ranks; value = numbers consumed by all ranks / time.
    Checked: the reduced counters hold exactly the job's pairs and numbers,
    and pi-hat lies within 5 sigma of pi."""
    import math

    import torch.distributed as tdist

    from paper_1112_5239_b200 import dist as D

    ws = tdist.get_world_size() if tdist.is_available() and tdist.is_initialized() else 1
    rk = tdist.get_rank() if ws > 1 else 0
    S, n = 2**20, 1024
    first, n_local = D.shard_range(S * ws, ws, rk)
    g = P.ChaoticPRNG(W.SEEDS[0], S * ws, P.V1, shard=(first, n_local))
    acc = torch.zeros(P.N_STATS, dtype=torch.int64, device=dev)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device=dev)

    def step():
        stats.zero_()
        g.consume(n, stats)
        D.allreduce_sum_(stats)
        acc.add_(stats)

    s = timed(step, calls)  # 3 warm-up + `calls` timed steps, all accumulated
    # verification (untimed): the fixed C5 stream space (2^23 streams, n =
    # 1024, one call) consumed sharded over however many ranks run, counters
    # SUM-all-reduced -- their sha256 is the same at every GPU count
    import hashlib

    c5 = W.CONFIGS["C5"]
    vstats = D.sharded_consume(W.SEEDS[0], c5["n_streams"], P.V1, c5["n"], 1)
    vsha = hashlib.sha256(P.as_u64(vstats).tobytes()).hexdigest()
    t = torch.tensor([s], dtype=torch.float64, device=dev)
    if ws > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    s = float(t.item())
    g.close()
    st = P.as_u64(acc)
    steps = calls + 3
    pairs, inside = int(st[1]), int(st[0])
    p = math.pi / 4
    sigma = 4 * math.sqrt(p * (1 - p) / pairs)
    return {"value": S * ws * n / s, "unit": UNIT, "ms_per_call": s * 1e3, "n_gpus": ws,
            "global_streams": S * ws, "n": n, "collective": "all_reduce SUM of 258 u64 per call "
            + (f"({tdist.get_backend()})" if ws > 1 else "(no-op at 1 GPU)"),
            "pairs_exact": pairs == steps * S * ws * n // 2,
            "hist_total_exact": int(st[2:].sum()) == steps * S * ws * n,
            "pi_hat": 4 * inside / pairs, "pi_within_5_sigma": abs(4 * inside / pairs - math.pi) < 5 * sigma,
            **_hist_chi2(st[2:]),
            "verify": {"streams": c5["n_streams"], "n": c5["n"], "calls": 1,
                       "stats_sha256": vsha, "note": "fixed global stream space; identical at every GPU count"}}


def measure_c1(P, torch, dev, with_oracle: bool) -> dict:
    """C1 (BASELINE configs[0]): V0 with `paper_defaults` --
    Listing 1 exactly (x = 123123123, Marsaglia's seeds) -- ONE
    stream, 10^6 outputs per call.  The stream is split over the whole GPU
    (csrc/v0_jump.cu): GF(2) jump-ahead of Listing 1's three xorshift
    generators to 128 x 148 segment starts plus an XOR scan of x; the same
    words as the one-thread chain, which is timed beside it
    (CIPRNG_V0_JUMP=0).  Calls continue the stream (state carried); the
    first call builds the jump plan (host polynomials, cached per shape) and
    is reported separately.  The oracle (single host core, same workload) is
    timed beside it and its words compared with the GPU's; the paper ran
    Listing 1 at 138 MS/s on one Xeon core."""
    n = 10**6
    stream = torch.cuda.current_stream()

    def run(env_jump: str, reps: int):
        old = os.environ.get("CIPRNG_V0_JUMP")
        os.environ["CIPRNG_V0_JUMP"] = env_jump
        try:
            g = P.ChaoticPRNG(0, 1, P.V0, paper_defaults=True)
        finally:
            if old is None:
                os.environ.pop("CIPRNG_V0_JUMP", None)
            else:
                os.environ["CIPRNG_V0_JUMP"] = old
        out = torch.empty((1, n), dtype=torch.int32, device=dev)
        a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a0.record(stream)
        g.generate(n, out=out)                   # call 1: plan + the parity call
        b0.record(stream)
        torch.cuda.synchronize()
        first_wall = time.perf_counter() - t0
        first = P.as_u32(out.cpu()).copy()
        path = int(g.info().store_path)
        for _ in range(3):
            g.generate(n, out=out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            g.generate(n, out=out)
        b.record(stream)
        torch.cuda.synchronize()
        g.close()
        return a.elapsed_time(b) / 1e3 / reps, a0.elapsed_time(b0), first_wall, first, path

    s, first_ms, first_wall, first, path = run("1", 200)
    s_seq, _, _, first_seq, _ = run("0", 3)
    row = {"value": n / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": 1, "n": n,
           "path": "jump-ahead (csrc/v0_jump.cu)" if path == 3 else f"store path {path}",
           "first_call_ms_device": first_ms, "first_call_s_wall_incl_plan": first_wall,
           "one_thread_chain": {"value": n / s_seq, "ms_per_call": s_seq * 1e3,
                                "bit_exact_vs_jump": bool(np.array_equal(first, first_seq))},
           "note": "one V0 stream over the whole GPU: jump-ahead to 128 x 148 segment starts, XOR scan of x; "
                   "back-to-back calls continue the stream (4 MB of output, L2-resident)",
           "paper_context": {"listing1_one_xeon_core_numbers_per_s": 1.38e8, "source": "PAPER.md P:1040-1041"}}
    if with_oracle:
        import oracle as O

        st = O.init_states(P.V0, 0, 0, 1, paper_defaults=True)
        t0 = time.perf_counter()
        ref = O.generate(P.V0, st, n)
        el = time.perf_counter() - t0
        row["cpu_baseline"] = {"value": n / el, "unit": UNIT, "cores": 1, "cpu_model": cpu_model(),
                               "kind": "oracle", "sample": "the whole C1 call (10^6 Listing-1 steps), once",
                               "bit_exact_vs_gpu": bool(np.array_equal(ref.reshape(-1), first.reshape(-1)))}
    return row


def measure_c4_sharded(P, torch, dev):
    """C4 (BASELINE configs[3]) as a job over every rank: V1, 2^23 streams x
    256 numbers x 466 calls = 1,000,727,379,968 numbers, the stream space
    split over the ranks (dist.shard_range: rank r owns a contiguous range
    of whole 32-stream groups) -- strong scaling, no collective on the data
    path.  (1) Throughput: the rank's 466 calls back to back (each call's
    output, 8 GiB / N, exceeds L2), CUDA events on the launching stream, max
    over ranks; value = all numbers / that time.  (2) Verification (untimed):
    a fresh handle regenerates the shard and digests every call on device
    (prng_digest: position-aware, additive across shards); the 466 per-call
    digests are SUM-all-reduced once, so the list -- and its sha256 -- is the
    same at every GPU count."""
    import hashlib

    import torch.distributed as tdist

    from paper_1112_5239_b200 import dist as D

    ws = tdist.get_world_size() if tdist.is_available() and tdist.is_initialized() else 1
    rk = tdist.get_rank() if ws > 1 else 0
    c4 = W.CONFIGS["C4"]
    S, n, calls = c4["n_streams"], c4["n"], c4["calls"]
    first, n_local = D.shard_range(S, ws, rk)
    out = torch.empty((n_local, n), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    g = P.ChaoticPRNG(W.SEEDS[0], S, P.V1, shard=(first, n_local))
    for _ in range(3):  # warm-up on a separate handle (state advanced; not verified)
        g.generate(n, out=out)
    a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    a_ev.record(stream)
    for _ in range(calls):
        g.generate(n, out=out)
    b_ev.record(stream)
    torch.cuda.synchronize()
    g.close()
    t = torch.tensor([a_ev.elapsed_time(b_ev) / 1e3], dtype=torch.float64, device=dev)
    if ws > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    sec = float(t.item())
    g = P.ChaoticPRNG(W.SEEDS[0], S, P.V1, shard=(first, n_local))
    acc = torch.zeros(calls, dtype=torch.int64, device=dev)
    for c in range(calls):
        g.generate(n, out=out)
        P.digest(out, first_stream=first, acc=acc[c:c + 1])
    g.close()
    D.allreduce_sum_(acc)
    dl = P.as_u64(acc)
    numbers = S * n * calls
    return {"value": numbers / sec, "unit": UNIT, "seconds": sec, "n_gpus": ws, "numbers": numbers,
            "streams": S, "n": n, "calls": calls, "scaling": "strong",
            "per_gpu_value": numbers / sec / ws,
            **_c4_write_fracs(numbers / sec / ws),
            "digests_first3": [int(v) for v in dl[:3]],
            "digest_list_sha256": hashlib.sha256(dl.tobytes()).hexdigest()}


def measure_curand(torch, dev, timed) -> dict:
    """Same-box context ("cuRAND ... not a target"): NVIDIA's
    library generators filling the C2-sized buffer (2^27 u32 = 512 MiB per
    call, curandGenerate) with the secondary rows' timing (L2 flushed before
    every call, CUDA events).  A LIBRARY on this box, not part of the path:
    the V1 row to set it against is `v1_c2_same_timing` (the headline kernel
    through the same helper)."""
    import ctypes

    lib = None
    for name in ("libcurand.so.10", "/usr/local/cuda/lib64/libcurand.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if lib is None:
        return {"unavailable": "libcurand not found"}
    words = 2**27
    out = torch.empty(words, dtype=torch.int32, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    rows = {}
    for name, rng in (("XORWOW", 101), ("PHILOX4_32_10", 161), ("MRG32K3A", 121), ("MTGP32", 141)):
        g = ctypes.c_void_p()
        if lib.curandCreateGenerator(ctypes.byref(g), rng) != 0:
            rows[name] = {"unavailable": "curandCreateGenerator failed"}
            continue
        lib.curandSetStream(g, st)
        lib.curandSetPseudoRandomGeneratorSeed(g, ctypes.c_ulonglong(W.SEEDS[0]))
        ptr = ctypes.c_void_p(out.data_ptr())

        def call():
            if lib.curandGenerate(g, ptr, ctypes.c_size_t(words)) != 0:
                raise RuntimeError(f"curandGenerate({name}) failed")

        s = timed(call, 20)
        rows[name] = {"value": words / s, "unit": UNIT, "ms_per_call": s * 1e3, "write_gbs": words * 4 / s / 1e9}
        lib.curandDestroyGenerator(g)
    del out
    return {"kind": "library context (not a target, not our path)", "words_per_call": words, "generators": rows}


def measure_secondary(P, torch, dev, args):
    """Other rows of SURVEY s8(a) on this GPU (not the headline): V2 store
    (C3), V0 store and V1 fused consumer; numbers/s with CUDA events."""
    res = {}
    stream = torch.cuda.current_stream()

    flush = L2Flush(torch, dev)

    def timed(fn, steps):
        """mean seconds per call; L2 flushed (untimed) before every call."""
        for _ in range(3):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for k in range(steps):
            flush(k)
            ev[k][0].record(stream)
            fn()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev) / 1e3 / steps

    if args.c5_only:
        return {"c5_consume_allreduce": measure_c5_sharded(P, torch, dev, timed)}
    res["c1_v0"] = measure_c1(P, torch, dev, with_oracle=not args.no_cpu_baseline)
    if args.c4_only:
        return {"c4_sharded_1e12": measure_c4_sharded(P, torch, dev)}
    S, n = W.CONFIGS["C3"]["n_streams"], W.CONFIGS["C3"]["n"]
    g = P.ChaoticPRNG(W.SEEDS[0], S, P.V2)
    out = torch.empty((S, n), dtype=torch.int32, device=dev)
    s = timed(lambda: g.generate(n, out=out), 20)
    # V2 is bound by the heavy FMA sub-pipe: each Barrett squaring needs IMAD +
    # IMAD.HI + IMAD = 8 heavy cycles per warp (IMAD.HI half rate)
    sq_peak = 148 * 4 * 32 * 1.965e9 / 8
    res["c3_v2_store"] = {"value": S * n / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S, "n": n,
                          "bbs_squarings_per_s": 12 * S * n / s,
                          "write_gbs_achieved": S * n * 4 / s / 1e9,  # the write BW actually achieved
                          "heavy_fma_model": {"peak_squarings_per_s": sq_peak,
                                                 "frac": 12 * S * n / s / sq_peak}}
    g.close()
    S0, n0 = 2**20, 128
    g = P.ChaoticPRNG(W.SEEDS[0], S0, P.V0)
    out = torch.empty((S0, n0), dtype=torch.int32, device=dev)
    s = timed(lambda: g.generate(n0, out=out), 20)
    res["v0_store"] = {"value": S0 * n0 / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S0, "n": n0}
    g.close()
    del out
    for name, var in (("v3_store", P.V3), ("v4_store", P.V4)):
        g = P.ChaoticPRNG(W.SEEDS[0], S0, var)
        out = torch.empty((S0, n0), dtype=torch.int32, device=dev)
        s = timed(lambda: g.generate(n0, out=out), 20)
        res[name] = {"value": S0 * n0 / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S0, "n": n0}
        g.close()
        del out
    S5, n5 = 2**20, 1024
    g = P.ChaoticPRNG(W.SEEDS[0], S5, P.V1)
    stats = torch.zeros(P.N_STATS, dtype=torch.int64, device=dev)
    s = timed(lambda: g.consume(n5, stats), 10)
    st5 = P.as_u64(stats)
    res["c5_v1_consume"] = {"value": S5 * n5 / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S5, "n": n5,
                            "pi_hat": 4 * int(st5[0]) / int(st5[1]), **_hist_chi2(st5[2:])}
    g.close()
    # the other variants in consumer mode (SURVEY s8(d) C5 "also V0 and V2"):
    # the like-for-like rows for the paper's no-store figures -- V3 is its
    # "optimized" xor64 kernel, V0 its naive Listing 1, V2 its BBS kernel
    for name, var in (("c5_v0_consume", P.V0), ("c5_v2_consume", P.V2), ("c5_v3_consume", P.V3)):
        g = P.ChaoticPRNG(W.SEEDS[0], S5, var)
        st5 = torch.zeros(P.N_STATS, dtype=torch.int64, device=dev)
        s = timed(lambda: g.consume(n5, st5), 10)
        res[name] = {"value": S5 * n5 / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S5, "n": n5,
                     "numbers_counted_exact": int(P.as_u64(st5)[2:].sum()) == 13 * S5 * n5}
        if var == P.V2:
            res[name]["heavy_fma_model"] = {"peak_squarings_per_s": sq_peak, "frac": 12 * S5 * n5 / s / sq_peak}
        g.close()
    res["c5_consume_allreduce"] = measure_c5_sharded(P, torch, dev, timed)
    from paper_1112_5239_b200 import battery as B

    g = P.ChaoticPRNG(W.SEEDS[0], S5, P.V1)
    bstats = torch.zeros(P.N_BATTERY, dtype=torch.int64, device=dev)
    s = timed(lambda: g.battery(n5, bstats), 10)
    pv = B.pvalues(P.as_u64(bstats), S5 * 13, n5)  # 3 warm-up + 10 timed calls
    res["v1_battery"] = {"value": S5 * n5 / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": S5, "n": n5,
                         "numbers_tested": S5 * n5 * 13, "pvalues": pv, "pass_1e-4": B.passes(pv)}
    g.close()
    # NEXT-3: batch chaotic Blum-Goldwasser encryption, 2^18 messages x 1024
    # units, moduli ~2^62 (a pool of 256 seeded Blum-prime keys), r < p, q
    from paper_1112_5239_b200 import bg as BGm

    import numpy as np

    gen = W.rng(99)
    keys = W.bg_keys(gen, 256, 31)
    Bm, Lm = 2**18, 1024
    Ns = np.array([keys[k % 256][2] for k in range(Bm)], dtype=np.uint64)
    rs = gen.integers(2, 2**30, Bm).astype(np.uint64)
    Nt = torch.from_numpy(Ns.view(np.int64)).to(dev)
    rt = torch.from_numpy(rs.view(np.int64)).to(dev)
    S0 = torch.from_numpy(gen.integers(0, 32, Bm).astype(np.int32)).to(dev)
    msg = torch.randint(0, 256, (Bm, Lm), dtype=torch.uint8, device=dev)
    s = timed(lambda: BGm.encrypt(True, Nt, rt, msg, S0), 10)
    res["cbg_encrypt"] = {"value": Bm * Lm / s, "unit": "keystream units/s", "ms_per_call": s * 1e3,
                          "messages": Bm, "units_per_message": Lm, "modulus_bits": 62, "unit_bits": 5}
    del msg
    # NEXT-4: Algorithm 1 (single-cell chaotic iterations, f = vectorial
    # negation on 32 cells, b = 8 -> 10..17 updates per output), 2^20 streams
    from paper_1112_5239_b200 import chaos as CH

    Sa, na = 2**20, 64
    za = torch.from_numpy(gen.integers(1, 2**31, Sa).astype(np.int32)).to(dev)
    xa = torch.zeros(Sa, dtype=torch.int32, device=dev)
    s = timed(lambda: CH.alg1_generate(32, 8, za, xa, na), 10)
    res["alg1_negation_b8"] = {"value": Sa * na / s, "unit": UNIT, "ms_per_call": s * 1e3, "streams": Sa,
                               "n": na, "cells": 32, "b": 8}
    # the headline kernel through the same helper (flushed, not charged) for the cuRAND comparison
    S2, n2 = W.CONFIGS["C2"]["n_streams"], W.CONFIGS["C2"]["n"]
    g = P.ChaoticPRNG(W.SEEDS[0], S2, P.V1)
    out = torch.empty((S2, n2), dtype=torch.int32, device=dev)
    s = timed(lambda: g.generate(n2, out=out), 20)
    res["v1_c2_same_timing"] = {"value": S2 * n2 / s, "unit": UNIT, "ms_per_call": s * 1e3,
                                "note": "event-timed, L2 flushed before each call, deferred write-back not charged"}
    g.close()
    del out
    res["curand_context"] = measure_curand(torch, dev, timed)
    # last: the 10^12-number job runs the GPU hot for seconds (power cap),
    # which slowed the row measured right after it by up to 13 % (r2b battery)
    res["c4_sharded_1e12"] = measure_c4_sharded(P, torch, dev)
    return res


def maybe_self_launch(args) -> int | None:
    """`--gpus N` (N > 1) outside torchrun: re-run this script under
    torch.distributed.run with N processes on this node (one per GPU, NCCL,
    rendezvous on 127.0.0.1) and return its exit code.  None = run here."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return None
    import socket
    import subprocess

    backend = os.environ.get("CIPRNG_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        import torch

        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs for NCCL, found {have}\n")
            return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--store-path", type=int, default=0, help="0 auto, 1 direct STG, 2 TMA tiles")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--c5-only", action="store_true", help="secondary rows: only the sharded C5 consume + all-reduce")
    ap.add_argument("--c4-only", action="store_true", help="secondary rows: only the sharded C4 10^12-number job")
    ap.add_argument("--streams", type=int, default=0, help="experiment override of streams per GPU")
    ap.add_argument("--rounds", type=int, default=0, help="experiment override of numbers per stream")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rc = maybe_self_launch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
