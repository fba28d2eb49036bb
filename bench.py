#!/usr/bin/env python
"""DGSM build + query benchmark (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dgsm|reference] [--config 2]

A step is one pass of the whole hot path (SURVEY.md §8(a) rows a1-a6 + a8) over
one synthetic frame: dgsm_build_plan + dgsm_build_run (project, scan, duplicate,
onesweep sort, ranges, accumulate + exp) + dgsm_query over the receivers.

* value  = Gaussian-ray evaluations per second of the whole step,
           64 * P (texel x listed Gaussian pairs, K shells each) / step time,
           inputs resident in HBM; L2 flushed (256 MiB write) before every step.
* e2e    = the same metric through the public API with the step's inputs copied
           from pinned host memory and T_out copied back inside the timed region.
* roofline = the accumulation kernel (a6, dominant), timed live with CUDA
           events recorded by the library around its launch; algorithmic FP32
           work per launch from an instrumented (untimed) run.
* cpu_baseline = the oracle (oracle/, fp64 C, all host cores) on a bounded
           sample: full binning + every s-th tile accumulated.
N > 1 (torchrun, or bench.py spawns it when WORLD_SIZE is unset): cfg1/2/4 weak
scaling — every rank builds and queries its own frame (independent light, no
data-path collective); cfg3/cfg5 strong scaling through distributed.StrongStep
(--layout light | shells | gaussian); every line also carries the cfg5 strong-
scaling run on the same N GPUs (strong_cfg5).  Time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2601_01660_b200 import synth  # noqa: E402  (seeded inputs only: no method arithmetic)

METRIC = "DGSM build Gaussian-ray evals/s and query Gaussians/s at 1/2/4/8 B200"
UNIT = "Gaussian-ray evals/s"

# Roofline numerator of the a6 accumulation: SURVEY.md §8(d)'s per-unit figure for
# the saturation-aware evaluation of one Gaussian-ray pair (texel x listed Gaussian,
# all K shells): ~70 FP32 ops + ~4 MUFU ops (FMA = 1 op), i.e. 74 ops per pair,
# times the 64 * P pairs one launch processes.
OPS_PER_PAIR_SURVEY = 74
# Work actually needed per pair class (informational): every pair
# 31 (delta-form test), live pair +30, window shell +16, saturated step +3.
OPS_PAIR = 31
OPS_LIVE = 30
OPS_SHELL = 16
OPS_STEP = 3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dgsm", choices=["dgsm", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0, help="shrink the scene (debug only)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle sample time")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-transfer", action="store_true", help="skip the NEXT-4 transfer timing")
    ap.add_argument("--no-strong", action="store_true", help="skip the cfg5 strong-scaling sub-record")
    ap.add_argument("--no-sequence", action="store_true", help="skip the cfg4 120-frame sequence sub-record")
    ap.add_argument("--no-graph", action="store_true", help="time the cfg1/2/4 step as stream launches "
                                                             "instead of a CUDA graph replay")
    ap.add_argument("--layout", default="auto", choices=["auto", "light", "shells", "gaussian"],
                    help="multi-GPU layout of cfg3/cfg5 (distributed.plan_layout)")
    return ap.parse_args()


def workload(cfg: int, scale: float, rank: int):
    from paper_2601_01660_b200 import synth
    if cfg == 2:
        s = synth.config2(scale=scale)
    elif cfg == 1:
        s = synth.config1()
    elif cfg == 4:
        s = synth.config4(frame=rank % 120, scale=scale)
    else:
        s = synth.make_config(cfg, scale=scale)
    if rank and cfg != 4:
        # weak scaling: an independent frame per rank (light moved by 5 cm per rank)
        lp = s.lights["position"].copy()
        lp[:, 0] += 0.05 * rank
        s.lights = dict(position=lp, t_max=s.lights["t_max"] + np.float32(0.05 * rank))
    return s


def cfg_desc(s, cfg):
    return {"workload": f"cfg{cfg}: {s.note}", "n_gaussians": s.n, "n_lights": s.L,
            "atlas": f"{s.res}x{s.res}x{s.K}", "queries": int(s.queries.shape[0]),
            "l2": "flushed before every step (256 MiB write)", "data": "synthetic, seeded (synth.py)"}


def query_roofline(ms: float, m: int, L: int, peaks: dict, ms_raw: float = None, cfg: int = 2, scale: float = 1.0):
    """a8 against HBM: algorithmic bytes and the sector-realistic
    count of a random-order gather (each row of taps is its own 32-B sector).
    ms: receivers in the scene's spatial (Morton) order; ms_raw: as generated."""
    peak = float(peaks.get("hbm_gbs", 7700.0))
    alg = m * (16 + 32 * L) * 1.0
    sec = m * (16 + 128 * L) * 1.0
    ach = alg / (ms * 1e-3) / 1e9
    out = {"kernel": "k_query (a8)", "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
           "frac": ach / peak, "alg_bytes_per_query": 16 + 32 * L,
           "alg_def": "SURVEY §8(d): 12 B position + 4 B T + 8 x 4 B taps per light",
           "sector_bytes_per_query": 16 + 128 * L,
           "sector_frac": sec / (ms * 1e-3) / 1e9 / peak,
           "peak_src": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "B200_PROFILING.md 7.7 TB/s",
           "timing": "L2 flushed before each launch, CUDA events, host launch overhead excluded",
           "receivers": "Morton-ordered scene receivers",
           "traffic": profiled_traffic("query_traffic.json", cfg, scale)}
    if ms_raw is not None:
        out["raw_order_frac"] = alg / (ms_raw * 1e-3) / 1e9 / peak
    return out


def transfer_timing(dev, n: int = 150_000, d: int = 3):
    """NEXT-4 SH lighting transfer (not part of the step): n avatar Gaussians
    (ActorsHQ scale, SURVEY cfg4) x the 64 x 128 lat-long grid, degree-3 probe,
    q = 1; L2 flushed, device time; 8 FP32 ops per (Gaussian, direction)."""
    import torch
    from paper_2601_01660_b200 import dgsm
    rng = np.random.default_rng(4)
    nr = rng.normal(size=(n, 3))
    nr /= np.linalg.norm(nr, axis=1, keepdims=True)
    nr = torch.from_numpy(nr.astype(np.float32)).to(dev)
    col = torch.from_numpy(rng.random((n, 3)).astype(np.float32)).to(dev)
    A = rng.normal(0, 0.5, (3, (d + 1) ** 2)).astype(np.float32)
    A[:, 0] = 2.5
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for _ in range(3):
        dgsm.sh_transfer(A, d, nr, col)
    ts = []
    for _ in range(10):
        flush.zero_()
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dgsm.sh_transfer(A, d, nr, col)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    ops = n * 64 * 128 * 8
    peak = torch.cuda.get_device_properties(dev).multi_processor_count * 128 * 1965e6 / 1e12
    return {"workload": f"{n} avatar Gaussians x 64x128 directions, SH degree {d}, q=1", "ms": ms,
            "gaussians_per_s": n / (ms * 1e-3), "gpu_launches": 3,
            "roofline": {"bound": "alu", "achieved": ops / (ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                         "frac": ops / (ms * 1e-3) / 1e12 / peak,
                         "alg_def": "8 FP32 ops per (Gaussian, direction): <w,n> 3, max 1, 4 FMA"}}


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        """Start sampling every 20 ms; return once nvidia-smi has produced its first
        sample (its start-up takes the driver lock and must not land in the timing)."""
        import threading
        self.lines = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.perf_counter(), line))
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 10.0:
            time.sleep(0.01)
        time.sleep(0.05)

    def mark(self):
        return time.perf_counter()

    def stop(self, t_begin=None, t_end=None):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=10)
        except Exception:
            pass
        self.thread.join(timeout=2)
        sel = [l for (t, l) in self.lines if (t_begin is None or t >= t_begin) and (t_end is None or t <= t_end + 0.03)]
        if not sel:  # timed region shorter than one sample period: nearest samples
            sel = [l for (_, l) in self.lines[-3:]]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in sel:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0])); smax = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ oracle legs
def oracle_sample(s, seconds: float, threads: int):
    """Oracle culled build of the scene: full binning + every stride-th tile.
    Returns dict(value evals/s, seconds, evals, stride)."""
    from oracle import oracle

    def run(stride):
        t0 = time.perf_counter()
        _, P, ev = oracle.build(s.gaussians, s.lights, s.res, s.K, tile_stride=stride, n_threads=threads,
                                return_evals=True)
        return time.perf_counter() - t0, P, ev

    n_items = s.L * (s.res // 8) ** 2
    # two pilots separate the fixed binning cost from the per-evaluation cost
    t1, P, ev1 = run(n_items)
    t2, _, ev2 = run(max(1, n_items // 64))
    per_eval = max(t2 - t1, 1e-6) / max(ev2 - ev1, 1)
    t_bin = max(t1, 0.0)
    acc_budget = max(seconds - t_bin, t_bin, 1.0)
    want = acc_budget / per_eval
    total_evals = 64.0 * P
    stride = int(max(1, min(n_items, round(total_evals / max(want, 1.0)))))
    dt, P, ev = run(stride)
    return {"value": ev / dt, "seconds": dt, "evals": ev, "stride": stride, "P": P,
            "est_full_build_s": t_bin + per_eval * total_evals}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    s = workload(args.config, args.scale, 0)
    thr = cores()
    budget = max(1.0, 150.0 / max(1, args.steps + args.warmup))
    vals, evs, secs, stride = [], 0, 0.0, None
    pilot = oracle_sample(s, budget, thr)
    stride = pilot["stride"]
    from oracle import oracle
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _, P, ev = oracle.build(s.gaussians, s.lights, s.res, s.K, tile_stride=stride, n_threads=thr,
                                return_evals=True)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            evs += ev; secs += dt
    value = evs / secs
    sample = (f"cfg{args.config}: full oracle binning of all {P} keys + Eq.3 accumulation on every "
              f"{stride}-th (light, tile) ({evs // max(args.steps, 1)} evals per step)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": cfg_desc(s, args.config),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
PAPER_CONTEXT = {
    "build_s_per_frame": {"roi_and_light_space_culling": 0.13, "no_light_space_culling": 17.1,
                          "no_roi_culling": 29.1},
    "hardware": "NVIDIA A100", "source": "PAPER.md:335 (§4.4 ablation D), 'across 5 scenes'",
    "note": "context only: other hardware; atlas size, K, occluder counts not stated by the paper",
}


class Ctx:
    """Process / device context of one rank."""

    def __init__(self, args):
        import torch
        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={self.world}")
        if not torch.cuda.is_available():
            sys.exit("bench.py: no CUDA device (the product arm has no CPU fallback)")
        if torch.cuda.device_count() < self.world and self.world > 1 and self.local >= torch.cuda.device_count():
            sys.exit(f"bench.py: rank {self.rank} needs GPU {self.local}, {torch.cuda.device_count()} visible")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.peaks = {}
        pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(pk):
            self.peaks = json.load(open(pk))
        self.n_sm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self.flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=self.dev)  # 256 MiB > 126 MB L2
        self.flush.zero_()  # first touch (page mapping) outside any timing

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()

    def max_over_ranks(self, x: float) -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return x
        t = torch.tensor([x], device=self.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def sum_over_ranks(self, x: float) -> float:
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return x
        t = torch.tensor([x], device=self.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t[0])


def fp32_peak(ctx):
    sm_mhz = float(ctx.peaks.get("sm_max_mhz", 1965.0))
    return ctx.n_sm * 128 * sm_mhz * 1e6 / 1e12, f"{ctx.n_sm} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (FMA = 1 op)"


def time_steps(step, K: int, warmup: int, ctx, sample_clocks: bool = True, acc_events: bool = True):
    """W untimed warm-up steps, then EXACTLY K timed steps, each after an L2 flush
    (outside the step's events), bracketed by barrier + synchronize; device time
    by CUDA events on the launching stream; the accumulation kernel's events are
    recorded by the library around its launch."""
    import torch
    from paper_2601_01660_b200 import dgsm
    for _ in range(warmup):
        ctx.flush.zero_()
        step()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    for e in ev:  # create the CUDA events now (torch creates them lazily on record)
        for x in e:
            x.record()
    torch.cuda.synchronize()
    sampler = ClockSampler(ctx.local)
    if sample_clocks:
        sampler.start()
    ctx.barrier()
    torch.cuda.synchronize()
    launches = 0
    wall0 = time.perf_counter()
    for i in range(K):
        e0, ea, eb, e1 = ev[i]
        ctx.flush.zero_()
        if acc_events:
            dgsm.set_accumulate_events(ea, eb)
        e0.record()
        launches += step()
        e1.record()
    dgsm.set_accumulate_events(None, None)
    torch.cuda.synchronize()
    wall1 = time.perf_counter()
    ctx.barrier()
    clocks = sampler.stop(wall0, wall1) if sample_clocks else None
    t_step = [ev[i][0].elapsed_time(ev[i][3]) for i in range(K)]
    t_acc = [ev[i][1].elapsed_time(ev[i][2]) for i in range(K)] if acc_events else None
    return {"t_step": t_step, "t_acc": t_acc, "launches": launches, "wall_ms": (wall1 - wall0) * 1e3,
            "clocks": clocks}


def time_fn(fn, reps: int, ctx):
    """Device time of fn() per call (median), L2 flushed before each; a ~0.2 ms
    device spin before the start event keeps the host's launch overhead out."""
    import torch
    ts = []
    for _ in range(reps):
        ctx.flush.zero_()
        torch.cuda._sleep(400_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def profiled_traffic(name, cfg, scale):
    """DRAM bytes per launch of a kernel from the committed ncu --set full capture
    (profiles/<name>, per config), or None when this workload was not captured."""
    prof = os.path.join(ROOT, "profiles", name)
    if not os.path.exists(prof) or abs(scale - 1.0) > 1e-9:
        return None
    try:
        return json.load(open(prof)).get(f"cfg{cfg}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def accumulate_roofline(st, acc_ms, ctx, cfg, scale):
    """a6 against the FP32 pipe: SURVEY §8(d)'s per-pair figure (frac) and the
    work the kernel actually does per pair class (work_frac)."""
    peak, peak_def = fp32_peak(ctx)
    alg_ops = OPS_PER_PAIR_SURVEY * st["pairs"]
    needed = OPS_PAIR * st["pairs"] + OPS_LIVE * st["pairs_live"] + OPS_SHELL * st["window_shells"] + OPS_STEP * st["steps"]
    achieved = alg_ops / (acc_ms * 1e-3) / 1e12
    traffic = profiled_traffic("accumulate_traffic.json", cfg, scale)
    return {"kernel": "k_accumulate (a6)", "bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "peak_def": peak_def, "frac": achieved / peak, "traffic": traffic, "alg_ops_per_launch": int(alg_ops),
            "alg_def": f"SURVEY §8(d): {OPS_PER_PAIR_SURVEY} FP32+MUFU ops per Gaussian-ray pair x {int(st['pairs'])} pairs",
            "work_ops_per_launch": int(needed),
            "work_frac": needed / (acc_ms * 1e-3) / 1e12 / peak,
            "work_def": (f"ops the kernel needs per pair class (DESIGN.md §6): {OPS_PAIR} per pair, +{OPS_LIVE} per live "
                         f"pair, +{OPS_SHELL} per window shell, +{OPS_STEP} per saturated step")}


def build_stats(dgsm, g, lights, res, K):
    """Instrumented (untimed) build: the accumulation's work counters and P."""
    sp = dgsm.BuildPlan(g, lights, res, K, dgsm.Options(collect_stats=True))
    sp.run()
    st = sp.stats()
    P = sp.n_keys
    del sp
    return st, P


def order_receivers(dgsm, xq, ctx):
    """Spatially coherent layout of the static scene receivers (done once per
    scene, DESIGN.md §6 a8): the Morton permutation, its device time, and the
    receivers in that order."""
    order = dgsm.receiver_order(xq)
    ms = time_fn(lambda: dgsm.receiver_order(xq, out=order), 3, ctx)
    return order.long(), ms


def cpu_baseline_line(s, cfg, seconds):
    cb = oracle_sample(s, seconds, cores())
    return {"value": cb["value"], "unit": UNIT, "cores": cores(), "kind": "oracle",
            "sample": f"cfg{cfg}: full oracle binning ({cb['P']} keys) + Eq.3 accumulation on every "
                      f"{cb['stride']}-th (light, tile): {cb['evals']} evals in {cb['seconds']:.1f} s; "
                      f"full oracle build estimated {cb['est_full_build_s']:.0f} s"}


# ----------------------------------------------------------- weak scaling
def weak_bench(args, ctx):
    """cfg1/2/4: every rank builds and queries its own frame (an independent
    light), no data-path collective; time = max over ranks."""
    import torch
    from paper_2601_01660_b200 import dgsm

    s = workload(args.config, args.scale, ctx.rank)
    g_host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in s.gaussians.items()}
    g = {k: v.to(ctx.dev) for k, v in g_host.items()}
    xq_raw = torch.from_numpy(np.ascontiguousarray(s.queries)).to(ctx.dev)
    order, order_ms = order_receivers(dgsm, xq_raw, ctx)
    xq = xq_raw[order].contiguous()
    q_host = xq.cpu().pin_memory()
    m = xq.shape[0]
    atlas = torch.empty((s.L, s.K, s.res, s.res), dtype=torch.float32, device=ctx.dev)
    T_out = torch.empty(m, dtype=torch.float32, device=ctx.dev)
    st, P = build_stats(dgsm, g, s.lights, s.res, s.K)
    # the per-frame entry point of a renderer: the sync-free build (no host
    # synchronisation inside the step) with a key capacity of 1.25 P, as a frame
    # stream would size it from an earlier frame; the status word is checked after
    cap = int(1.25 * P) + 4096
    builder = dgsm.AsyncBuilder(s.lights, s.res, s.K, s.n, cap, device=ctx.dev)

    def step():
        builder(g, atlas)  # dgsm_build_async: plan + run, no host sync
        nl = builder.launches
        dgsm.query(atlas, s.lights, xq, out=T_out)
        return nl + dgsm.last_launch_count()

    # stream launches: the accumulation kernel's duration per step (library events)
    r = time_steps(step, args.steps, args.warmup, ctx, sample_clocks=args.no_graph)
    launch_mode = "stream launches"
    r_stream_ms = float(np.mean(r["t_step"]))
    if not args.no_graph:
        # the step as a renderer runs it every frame: the sync-free build + query captured
        # once in a CUDA graph and replayed (same 21 kernels, same inputs in HBM; only the
        # host launch overhead and inter-kernel gaps go), L2 flushed before every replay
        gs = torch.cuda.Stream(ctx.dev)
        gs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(gs):
            step()
        torch.cuda.current_stream().wait_stream(gs)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            step()
        per_step = r["launches"] // args.steps

        def replay():
            graph.replay()
            return per_step

        t_acc = r["t_acc"]
        r = time_steps(replay, args.steps, args.warmup, ctx, acc_events=False)
        r["t_acc"] = t_acc
        launch_mode = "one CUDA graph replay per step (captured once from the stream-launched step)"
    bst = builder.status()
    if bst["overflow"] or bst["n_keys"] != P:
        sys.exit(f"bench.py: sync-free build status {bst} (expected {P} keys)")
    K = args.steps
    total_ms = float(np.sum(r["t_step"]))
    total_max = ctx.max_over_ranks(total_ms)
    units_all = ctx.sum_over_ranks(64.0 * P)
    value = units_all * K / (total_max * 1e-3)
    tq = time_fn(lambda: dgsm.query(atlas, s.lights, xq, out=T_out), K, ctx)
    tq_raw = time_fn(lambda: dgsm.query(atlas, s.lights, xq_raw, out=T_out), K, ctx)

    e2e = None
    if not args.no_e2e:
        T_host = torch.empty(m, dtype=torch.float32).pin_memory()
        fr = dgsm.FrameHost(s.lights, s.res, s.K, device=ctx.dev)
        for _ in range(2):
            fr(g_host, q_host, T_host)
        torch.cuda.synchronize()
        # frames back to back (the steady state of a frame stream): frame i+1's uploads
        # (copy stream) overlap frame i's build; time = the K-frame span minus the flushes
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fl = []
        e0.record()
        for i in range(K):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.flush.zero_()
            b.record()
            fl.append((a, b))
            fr(g_host, q_host, T_host)
        e1.record()
        torch.cuda.synchronize()
        te_ms = e0.elapsed_time(e1) - float(np.sum([a.elapsed_time(b) for a, b in fl]))
        # one isolated frame at a time (synchronised: no overlap with a neighbour)
        iso = []
        for i in range(K):
            ctx.flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fr(g_host, q_host, T_host)
            b.record()
            torch.cuda.synchronize()
            iso.append(a.elapsed_time(b))
        te_fh = ctx.max_over_ranks(te_ms)
        # dgsm.FrameStream (the frame loop API): uploads on a copy stream gated on the
        # previous frame's accumulation, the sync-free build + query as one CUDA-graph
        # replay per buffer set, T back on a second copy stream; W warm-up frames, then
        # K frames back to back, each after an L2 flush (span minus the flushes)
        fs = dgsm.FrameStream(s.lights, s.res, s.K, s.n, m, cap, device=ctx.dev)
        Ts = [torch.empty(m, dtype=torch.float32).pin_memory() for _ in range(2)]
        for i in range(max(args.warmup, 2)):
            fs(g_host, q_host, Ts[i & 1])
        fs.wait()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fl = []
        e0.record()
        for i in range(K):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ctx.flush.zero_()
            b.record()
            fl.append((a, b))
            fs(g_host, q_host, Ts[i & 1])
        for ev_ in fs.ev_down:  # the last frames' T copies are inside the timed region
            torch.cuda.current_stream().wait_event(ev_)
        e1.record()
        torch.cuda.synchronize()
        fst = fs.status()
        if fst["overflow"] or fst["n_keys"] != P:
            sys.exit(f"bench.py: FrameStream build status {fst} (expected {P} keys)")
        te_max = ctx.max_over_ranks(e0.elapsed_time(e1) - float(np.sum([a.elapsed_time(b) for a, b in fl])))
        h2d = sum(v.numel() * 4 for v in g_host.values()) + q_host.numel() * 4
        e2e = {"value": units_all * K / (te_max * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(m * 4), "ms_per_step": te_max / K,
               "api": ("dgsm.FrameStream (host buffers in, T to a pinned host buffer): frames back to back, "
                       "frame i+1's receivers uploaded on a copy stream as soon as its buffer set is free and "
                       "its Gaussians from frame i's accumulation on, the build + query as one CUDA-graph "
                       "replay, T copied back on a second stream; K-frame span (up to the last T copy) minus "
                       "the L2 flushes"),
               "frame_host_ms_per_step": te_fh / K,
               "frame_host_value": units_all * K / (te_fh * 1e-3),
               "isolated_ms_per_frame": float(np.median(iso)),
               "isolated_value": units_all / (ctx.max_over_ranks(float(np.median(iso))) * 1e-3),
               "frame_host_api": ("dgsm_frame_host (one C call per frame: plan with its host sync, run, "
                                  "query): frames back to back, and isolated_* = one synchronised frame "
                                  "at a time")}
    acc_ms = float(np.mean(r["t_acc"]))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ctx.world, "steps": K, "warmup": args.warmup,
        "ms_per_step": total_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "dtype_note": "accumulation and query taps in fp32; binning geometry and query index math in fp64",
        "data": "synthetic",
        "config": dict(cfg_desc(s, args.config),
                       parallelism=f"{ctx.world} independent frame(s), one per rank, no data-path collective",
                       build=f"dgsm_build_async (no host sync), key capacity {cap} (1.25 P); status checked",
                       receivers=("scene receivers stored in Morton order (dgsm_receiver_order, once per scene: "
                                  f"{order_ms * 1e3:.0f} us)")),
        "launch_mode": launch_mode, "ms_per_step_stream_launches": r_stream_ms,
        "step_ms_each": [round(x, 3) for x in r["t_step"]], "step_ms_median": float(np.median(r["t_step"])),
        "wall_ms_per_step_incl_flush": r["wall_ms"] / K,
        "accumulate_ms": acc_ms, "accumulate_share": acc_ms / float(np.mean(r["t_step"])),
        "query_ms": tq, "query_ms_raw_order": tq_raw, "receiver_order_ms_once": order_ms,
        "query_gaussians_per_s": m / (tq * 1e-3) * ctx.world,
        "keys_P": int(P), "gaussian_ray_evals_per_step": int(64 * P),
        "accumulate_work": {k: int(v) for k, v in st.items()},
        "gpu_launches": int(r["launches"]),
        "roofline": accumulate_roofline(st, acc_ms, ctx, args.config, args.scale),
        "query_roofline": query_roofline(tq, m, s.L, ctx.peaks, tq_raw, args.config, args.scale),
        "clocks": r["clocks"], "paper_context": PAPER_CONTEXT,
    }
    if e2e:
        line["e2e"] = e2e
    return line, s


# --------------------------------------------------------- strong scaling
def strong_bench(cfg, steps, warmup, ctx, scale=1.0, layout_mode="auto", e2e=True, clocks=True):
    """cfg3/cfg5 over the node: distributed.StrongStep — the
    layout's sharded build (light-parallel, or Gaussian shards + one NCCL
    reduce-scatter + exp) and the sharded query (chunk query + all-reduce SUM of
    split lights + all-reduce PRODUCT).  Total work is fixed (strong scaling)."""
    import torch
    from paper_2601_01660_b200 import dgsm
    from paper_2601_01660_b200 import distributed as D

    s = synth.make_config(cfg, scale=scale)
    g_host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in s.gaussians.items()}
    g = {k: v.to(ctx.dev) for k, v in g_host.items()}
    xq_raw = torch.from_numpy(np.ascontiguousarray(s.queries)).to(ctx.dev)
    order, order_ms = order_receivers(dgsm, xq_raw, ctx)
    xq = xq_raw[order].contiguous()
    del xq_raw, order
    m = xq.shape[0]
    # LPT costs: per-light key counts P_l from one replicated plan (once per scene here;
    # per frame a renderer would reuse the previous frame's counts)
    plan = dgsm.BuildPlan(g, s.lights, s.res, s.K)
    ranges = plan.light_key_ranges()
    P_all = plan.n_keys
    del plan
    layout = D.plan_layout(s.L, ctx.world, s.K, D.light_costs(ranges), layout_mode)
    pgroups = D.make_groups(layout) if ctx.world > 1 else [None] * len(layout.groups)
    cache = {}
    step_obj = D.StrongStep(layout, pgroups, s.lights, s.res, D.cuda_build_fn(cache, s.res, s.K), D.cuda_exp_fn,
                            D.cuda_chunks_fn(s.res, s.K), D.cuda_combine_fn, ctx.dev)
    b = step_obj.builder
    if b.g > 1:
        s0, s1 = D.shard_range(s.n, b.idx, b.g)
    else:
        s0, s1 = 0, s.n
    g_mine = {k: v[s0:s1] for k, v in g.items()}
    st, P_mine = build_stats(dgsm, g_mine, b.sub, s.res, s.K)

    # launch count of one step on this rank (library counters, one untimed step):
    # the build, the exp epilogue (Gaussian shards), the chunk query, the combine
    step_obj(g, xq)
    j = layout.group_index(ctx.rank)
    split = layout.split_lights(j) if j >= 0 else []
    nl = (sum(cb[0].launches for cb in cache.values()) + (1 if b.g > 1 else 0) + 1
          + (1 if split and layout.groups[j][0] == ctx.rank else 0))

    def step_counted():
        step_obj(g, xq)
        return nl

    r = time_steps(step_counted, steps, warmup, ctx, sample_clocks=clocks)
    total_ms = float(np.sum(r["t_step"]))
    total_max = ctx.max_over_ranks(total_ms)
    value = 64.0 * P_all * steps / (total_max * 1e-3)
    acc_ms = float(np.mean(r["t_acc"]))
    acc_max = ctx.max_over_ranks(acc_ms)
    tq = time_fn(lambda: D.query_sharded(step_obj.atlas, s.lights, xq, layout, pgroups, step_obj.chunks_fn,
                                         step_obj.combine_fn, s.res), steps, ctx)
    tq = ctx.max_over_ranks(tq)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ctx.world, "steps": steps, "warmup": warmup,
        "ms_per_step": total_max / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "dtype_note": "accumulation and query taps in fp32; binning geometry and query index math in fp64",
        "data": "synthetic",
        "config": dict(cfg_desc(s, cfg), parallelism=(
            f"{ctx.world} rank(s), layout {layout.mode}: groups {layout.groups}, lights {layout.lights_of}"
            + (" (Gaussian shards + one NCCL reduce-scatter of tau over the group's (light, shell) planes + exp; "
               "query: chunk sums all-reduced, product all-reduced)" if max(len(x) for x in layout.groups) > 1
               else " (lights dealt by LPT on per-light key counts; no build communication; query product "
                    "all-reduced)")),
            receivers=f"Morton-ordered once per scene ({order_ms * 1e3:.0f} us)"),
        "step_ms_each": [round(x, 3) for x in r["t_step"]],
        "keys_P": int(P_all), "keys_P_per_light": [int(e - b_) for b_, e in ranges],
        "gaussian_ray_evals_per_step": int(64 * P_all),
        "accumulate_ms_rank0": acc_ms, "accumulate_ms_max": acc_max,
        "accumulate_share": acc_ms / float(np.mean(r["t_step"])),
        "query_ms": tq, "query_gaussians_per_s": m / (tq * 1e-3),
        "gpu_launches": int(r["launches"]),
        "roofline": accumulate_roofline(st, acc_ms, ctx, cfg, scale),
        "accumulate_work_rank0": {k: int(v) for k, v in st.items()},
        "query_roofline": query_roofline(tq, m, s.L, ctx.peaks, None, cfg, scale) if ctx.world == 1 else None,
        "clocks": r["clocks"],
    }
    if e2e:
        # this rank's inputs host -> device each step (its Gaussian range and all
        # receivers), the product T device -> host on rank 0, inside the timed region
        g_h = {k: v[s0:s1] for k, v in g_host.items()}
        g_d = {k: v[s0:s1] for k, v in g.items()}
        q_host = xq.cpu().pin_memory()
        T_host = torch.empty(m, dtype=torch.float32).pin_memory()
        te = []
        ctx.barrier()
        for i in range(steps):
            ctx.flush.zero_()
            a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for k_, v_ in g_h.items():
                g_d[k_].copy_(v_, non_blocking=True)
            xq.copy_(q_host, non_blocking=True)
            T = step_obj(g, xq)
            if ctx.rank == 0:
                T_host.copy_(T, non_blocking=True)
            bb.record()
            te.append((a, bb))
        torch.cuda.synchronize()
        te_ms = ctx.max_over_ranks(float(np.sum([a.elapsed_time(bb) for a, bb in te])))
        out["e2e"] = {"value": 64.0 * P_all * steps / (te_ms * 1e-3), "unit": UNIT,
                      "h2d_bytes_per_step": int(sum(v.numel() * 4 for v in g_h.values()) + m * 12),
                      "d2h_bytes_per_step": int(m * 4) if ctx.rank == 0 else 0, "ms_per_step": te_ms / steps,
                      "api": "torch copies (pinned host) + distributed.StrongStep (dgsm_build / exp / query_chunks)"}
    del cache, step_obj, g, g_mine
    torch.cuda.empty_cache()
    return out, s


# ------------------------------------------------ cfg4 animated sequence
def _seq_frame(f):
    from paper_2601_01660_b200 import synth as sy
    return sy.Config4Sequence.frame_static(f)


def sequence_frames(seq, frames):
    """The occluders (walking avatar + prop) of every frame, generated on the
    host before any timing (a process pool: ~0.3 s of numpy per frame)."""
    import concurrent.futures as cf
    import multiprocessing as mpc
    workers = max(1, min(16, cores()))
    with cf.ProcessPoolExecutor(max_workers=workers, mp_context=mpc.get_context("spawn")) as ex:
        return list(ex.map(_seq_frame, frames))


def sequence_bench(ctx, frames=None, warmup=3, modes=("full", "roi_slab")):
    """cfg4 as BASELINE defines it: 120 frames of the walking
    avatar + prop (the occluders of the paper's setting) over the static
    2 M-Gaussian room (the receivers, Morton-ordered once).  Per frame: the
    frame's occluders host -> device (pinned), the sync-free build
    (dgsm_build_async) and the query of all 2 M receivers, replayed from ONE
    CUDA graph (no host synchronisation inside a frame); in roi_slab mode the
    receiver-driven ROI slab (dgsm_active_slab) restricts the build
    first — the paper's own timed setting (0.13 s/frame on an A100).
    Per-frame device time by CUDA events, L2 flushed between frames."""
    import torch
    from paper_2601_01660_b200 import dgsm
    seq = synth.Config4Sequence()
    frames = list(range(seq.n_frames)) if frames is None else list(frames)
    occ = sequence_frames(seq, sorted(set(frames)))
    occ = dict(zip(sorted(set(frames)), occ))
    n = occ[frames[0]]["means"].shape[0]
    host = {f: {k: torch.from_numpy(v).pin_memory() for k, v in o.items()} for f, o in occ.items()}
    g = {k: v.to(ctx.dev) for k, v in host[frames[0]].items()}
    xq_raw = torch.from_numpy(seq.queries).to(ctx.dev)
    order, order_ms = order_receivers(dgsm, xq_raw, ctx)
    xq = xq_raw[order].contiguous()
    del xq_raw, order
    m = xq.shape[0]
    res, K, L = seq.res, seq.K, 1
    atlas = torch.empty((L, K, res, res), dtype=torch.float32, device=ctx.dev)
    T = torch.empty(m, dtype=torch.float32, device=ctx.dev)
    out = {"workload": f"cfg4: {len(frames)} frames, walking 150k avatar + 50k prop occluders over a 2M-Gaussian "
                       f"room (receivers), 1 light, {res}^2 x {K}",
           "frames": len(frames), "receivers": m, "occluders_per_frame": n,
           "receiver_order_ms_once": order_ms, "paper_context_s_per_frame": PAPER_CONTEXT["build_s_per_frame"],
           "api": "per frame: H2D of the occluders, then one CUDA-graph replay of dgsm_build_async + dgsm_query "
                  "(roi_slab: dgsm_active_slab first)"}
    slab = torch.empty(dgsm.lib().dgsm_slab_bytes(1, res), dtype=torch.uint8, device=ctx.dev)
    for mode in modes:
        opts = dgsm.Options(slab=slab) if mode == "roi_slab" else dgsm.Options()
        if mode == "roi_slab":
            dgsm.active_slab(xq, seq.roi(frames[0]), seq.lights, res, K, out=slab)
        # key capacity from a few frames' plans (the walk changes P slowly), with margin
        Ps = []
        for f in frames[:: max(1, len(frames) // 4)]:
            gd = dgsm.to_device({k: v.numpy() for k, v in host[f].items()}, ctx.dev)
            if mode == "roi_slab":
                dgsm.active_slab(xq, seq.roi(f), seq.lights, res, K, out=slab)
            Ps.append(dgsm.BuildPlan(gd, seq.lights, res, K, opts).n_keys)
        cap = int(1.5 * max(Ps)) + 4096
        ab = dgsm.AsyncBuilder(seq.lights, res, K, n, cap, opts, device=ctx.dev)
        side = torch.cuda.Stream(device=ctx.dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                ab(g, atlas)
                dgsm.query(atlas, seq.lights, xq, out=T)
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            ab(g, atlas)
            dgsm.query(atlas, seq.lights, xq, out=T)
        launches = ab.launches + 1
        status = torch.zeros((len(frames), 16), dtype=torch.uint8, device=ctx.dev)

        def frame(i, f):
            for k_, v_ in host[f].items():
                g[k_].copy_(v_, non_blocking=True)
            if mode == "roi_slab":
                dgsm.active_slab(xq, seq.roi(f), seq.lights, res, K, out=slab)
            graph.replay()
            status[i].copy_(ab.status_buf)

        for i in range(warmup):
            ctx.flush.zero_()
            frame(i % len(frames), frames[i % len(frames)])
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in frames]
        for a, b in ev:
            a.record(); b.record()
        torch.cuda.synchronize()
        for i, f in enumerate(frames):
            ctx.flush.zero_()
            ev[i][0].record()
            frame(i, f)
            ev[i][1].record()
        torch.cuda.synchronize()
        t = np.array([a.elapsed_time(b) for a, b in ev])
        st = status.cpu().numpy()
        nk = st[:, :8].copy().view(np.uint64).reshape(-1).astype(np.int64)
        over = st[:, 8:12].copy().view(np.uint32).reshape(-1)
        # frames back to back as a renderer streams them: frame i+1's occluders go up on a
        # copy stream into the other of two device buffer sets (one graph captured per set)
        # while frame i's graph runs; span minus the L2 flushes / frames
        g_b = {k_: torch.empty_like(v_) for k_, v_ in g.items()}
        graph_b = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            ab(g_b, atlas)
            dgsm.query(atlas, seq.lights, xq, out=T)
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(graph_b):
            ab(g_b, atlas)
            dgsm.query(atlas, seq.lights, xq, out=T)
        bufs, graphs = [g, g_b], [graph, graph_b]
        cs = torch.cuda.Stream(device=ctx.dev)
        ev_up = [torch.cuda.Event() for _ in range(2)]
        ev_free = [torch.cuda.Event() for _ in range(2)]
        cur = torch.cuda.current_stream()
        for e_ in ev_free:
            e_.record(cur)
        status_s = torch.zeros((len(frames), 16), dtype=torch.uint8, device=ctx.dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fl = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in frames]
        for a_, b_ in fl:
            a_.record(); b_.record()
        torch.cuda.synchronize()
        e0.record(cur)
        for i, f in enumerate(frames):
            kb = i & 1
            cs.wait_event(ev_free[kb])
            with torch.cuda.stream(cs):
                for k_, v_ in host[f].items():
                    bufs[kb][k_].copy_(v_, non_blocking=True)
                ev_up[kb].record(cs)
            fl[i][0].record(cur)
            ctx.flush.zero_()
            fl[i][1].record(cur)
            cur.wait_event(ev_up[kb])
            if mode == "roi_slab":
                dgsm.active_slab(xq, seq.roi(f), seq.lights, res, K, out=slab)
            graphs[kb].replay()
            ev_free[kb].record(cur)
            status_s[i].copy_(ab.status_buf)
        e1.record(cur)
        torch.cuda.synchronize()
        span = e0.elapsed_time(e1) - float(sum(a_.elapsed_time(b_) for a_, b_ in fl))
        st_s = status_s.cpu().numpy()
        nk_s = st_s[:, :8].copy().view(np.uint64).reshape(-1).astype(np.int64)
        over_s = st_s[:, 8:12].copy().view(np.uint32).reshape(-1)
        stream_rec = {"ms_per_frame": span / len(frames), "value": float(64.0 * nk_s.sum() / (span * 1e-3)),
                      "overflow_frames": int((over_s != 0).sum()),
                      "api": "frames back to back: occluder upload of frame i+1 on a copy stream into a second "
                             "buffer set (its own captured graph) while frame i's graph runs; span minus L2 flushes",
                      "vs_paper_s_per_frame": (PAPER_CONTEXT["build_s_per_frame"]["roi_and_light_space_culling"]
                                               / (span / len(frames) * 1e-3)) if mode == "roi_slab" else None}
        del graph_b
        out[mode] = {"ms_per_frame_mean": float(t.mean()), "ms_per_frame_p50": float(np.percentile(t, 50)),
                     "ms_per_frame_p99": float(np.percentile(t, 99)), "ms_total": float(t.sum()),
                     "value": float(64.0 * nk.sum() / (t.sum() * 1e-3)), "unit": UNIT,
                     "keys_P_min": int(nk.min()), "keys_P_max": int(nk.max()), "key_capacity": cap,
                     "overflow_frames": int((over != 0).sum()), "gpu_launches_per_frame": int(launches),
                     "h2d_bytes_per_frame": int(n * 44),
                     "vs_paper_s_per_frame": (PAPER_CONTEXT["build_s_per_frame"]["roi_and_light_space_culling"]
                                              / (t.mean() * 1e-3)) if mode == "roi_slab" else None,
                     "stream": stream_rec}
        del graph, ab
    torch.cuda.empty_cache()
    return out


def next_rows_bench(ctx, reps=3):
    """The NEXT rows measured on cfg4's frame 0 (the paper's own setting, one B200):
    f3 / ablation D — the unculled build, every Gaussian in every tile,
    against the light-space-culled build of the same occluders; f2 (P:L190,
    P:L308-317) — the footprint-averaged query of the 2 M room Gaussians (7-point
    stencil and 32 Monte Carlo samples) against the centre query.  Device time by
    CUDA events, L2 flushed before each call; medians of `reps`."""
    import torch
    from paper_2601_01660_b200 import dgsm
    seq = synth.Config4Sequence()
    res, K = seq.res, seq.K
    g = dgsm.to_device(seq.frame(0), ctx.dev)
    out = {"workload": f"cfg4 frame 0: {g['means'].shape[0]} occluders (avatar + prop), 1 light, {res}^2 x {K}; "
                       f"receivers = the {seq.room['means'].shape[0]} room Gaussians"}
    atlas = torch.empty((1, K, res, res), dtype=torch.float32, device=ctx.dev)
    for name, opts in (("culled", dgsm.Options()), ("unculled", dgsm.Options(tile_cull=False))):
        b = dgsm.Builder(seq.lights, res, K, opts, device=ctx.dev)
        b(g, atlas)
        ms = time_fn(lambda: b(g, atlas), reps, ctx)
        P = dgsm.BuildPlan(g, seq.lights, res, K, opts).n_keys
        out[f"build_{name}"] = {"ms": ms, "keys_P": int(P), "gaussian_ray_evals_per_s": 64.0 * P / (ms * 1e-3)}
        del b
        torch.cuda.empty_cache()
    out["ablation_d_slowdown"] = out["build_unculled"]["ms"] / out["build_culled"]["ms"]
    out["paper_ablation_d"] = {"culled_s": 0.13, "unculled_s": 17.1, "slowdown": 17.1 / 0.13,
                               "source": "PAPER.md:335 (A100, ROI + light-space culling vs no light-space culling)"}
    dgsm.Builder(seq.lights, res, K, device=ctx.dev)(g, atlas)
    rg = dgsm.to_device({k: seq.room[k] for k in ("means", "scales", "rotations")}, ctx.dev)
    m = rg["means"].shape[0]
    T = torch.empty(m, dtype=torch.float32, device=ctx.dev)
    fq = {"center": time_fn(lambda: dgsm.query(atlas, seq.lights, rg["means"], out=T), reps, ctx)}
    z7, w7 = dgsm.footprint_stencil("stencil7")
    zmc = synth.mc_offsets(32, 3)
    wmc = np.full(32, 1.0 / 32, np.float32)
    for name, (z, w) in (("stencil7", (z7, w7)), ("mc32", (zmc, wmc))):
        fq[name] = time_fn(lambda: dgsm.query_footprint(atlas, seq.lights, rg, z, w, out=T), reps, ctx)
    out["query_footprint_ms"] = fq
    out["query_footprint_receivers_per_s"] = {k: m / (v * 1e-3) for k, v in fq.items()}
    return out


def run_dgsm(args):
    import torch
    import torch.distributed as dist

    from paper_2601_01660_b200 import build_ext

    ctx = Ctx(args)
    if ctx.world > 1:
        dist.init_process_group("nccl", device_id=ctx.dev)
    if ctx.rank == 0:
        build_ext.build()
    ctx.barrier()
    strong = args.config in (3, 5)
    if strong:
        line, s = strong_bench(args.config, args.steps, args.warmup, ctx, args.scale, args.layout,
                               e2e=not args.no_e2e)
    else:
        line, s = weak_bench(args, ctx)
    if not args.no_sequence and args.config in (2, 4) and ctx.rank == 0:  # a single-GPU workload
        try:
            line["cfg4_sequence"] = sequence_bench(ctx)
        except Exception as e:  # reported, not fatal for the main line
            line["cfg4_sequence"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_sequence and args.config in (2, 4) and ctx.rank == 0:
        try:
            line["next_rows"] = next_rows_bench(ctx)
        except Exception as e:  # reported, not fatal for the main line
            line["next_rows"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if not args.no_strong and args.config == 2:
        # the strong-scaling configuration of BASELINE (cfg5) on the same N GPUs
        try:
            sub, _ = strong_bench(5, min(args.steps, 5), 3, ctx, 1.0, args.layout, e2e=False, clocks=False)
            line["strong_cfg5"] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "n_gpus", "scaling", "config",
                                                        "keys_P", "keys_P_per_light", "accumulate_ms_max",
                                                        "query_ms", "roofline", "step_ms_each")}
        except Exception as e:  # reported, not fatal for the main line
            line["strong_cfg5"] = {"error": f"{type(e).__name__}: {e}"[:300]}
    if ctx.rank == 0:
        if not args.no_transfer:
            line["transfer"] = transfer_timing(ctx.dev)
        if not args.no_cpu_baseline and ctx.world == 1:
            if 64 * line["keys_P"] <= 64 * 60_000_000:
                line["cpu_baseline"] = cpu_baseline_line(s, args.config, args.cpu_seconds)
            else:
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores(), "kind": "oracle",
                                        "sample": "skipped: the oracle's full binning of this many keys exceeds "
                                                  "the bounded sample (see the cfg2 line)"}
        print(json.dumps(line), flush=True)
    if ctx.world > 1:
        ctx.barrier()
        dist.destroy_process_group()


def spawn(args):
    """`bench.py --gpus N` without a torchrun environment: launch N ranks with
    torch.distributed.run on this node (127.0.0.1) and pass the line through."""
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if n < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n}")
    import socket
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn(args)
    run_dgsm(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
