#!/usr/bin/env python
"""FSBM collision-coalescence step benchmark (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config C2, BASELINE.json configs[1]): CONUS-12km-shaped grid
ni x nj x nk = 425 x 300 x 50 (6.375 M points), 33 bins, SURVEY 8(d)
"thunderstorm" input (all six hydrometeor categories populated at every
mask-true point, cloud fraction 1.0, seed 42), golovin tables (coeff 1,
level_scale 1.5, pair_scale_step 0.05), dt = 1 s, substeps = 1.

A step = one fissioned_step phase 2 (coal_step at every mask-true point) over the
rank's i-slab.  Multi-GPU: i-slabs are independent shards (column-local physics,
no halo); NCCL only all-reduces the end-of-step diagnostics.  The thunderstorm
state turns stiff after ~4 steps at dt=1, so every step starts from the same
input: the state is restored device-to-device (outside the per-step CUDA events)
before each step.  The state (10 GB) is ~80x the L2, so no extra flush is needed.

value      device time (CUDA events around each step call, summed, max over ranks)
e2e        same metric through the host C ABI fsbm_step_grid_host: H2D of the state
           + step + D2H, host buffers pinned
roofline   FP64 pipe: algorithmic 12 FLOP per active (pair,i,j) triple
           / the coal kernel's own CUDA-event time, against the FP64 DFMA roof
           measured live on this GPU (MEASURED_PEAKS.json has no FP64 figure)
cpu_baseline  the reference's fissioned_step (oracle/_ref, collapse-3 arena,
           on-demand, all host threads) on a bounded i-slab sample of the same bytes
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FSBM coalescence grid-point updates/sec (CONUS-12km shape, 33 bins) @1/2/4/8 B200"
UNIT = "grid-point updates/s"
CONFIG = dict(ni=425, nj=300, nk=50, nkr=33, cloud_fraction=1.0, seed=42, dt=1.0, substeps=1)
FLOP_PER_TRIPLE = 12


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--numerics", default="fast", choices=["fast", "exact"])
    ap.add_argument("--nkr", type=int, default=33)
    ap.add_argument("--ni", type=int, default=CONFIG["ni"])
    ap.add_argument("--nj", type=int, default=CONFIG["nj"])
    ap.add_argument("--nk", type=int, default=CONFIG["nk"])
    ap.add_argument("--cf", type=float, default=CONFIG["cloud_fraction"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank owns a full C2-shaped i-slab of an N x C2 domain "
                         "(stacked in i); strong: the C2 domain is split across ranks")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 4 + k and r[4 + k].lower().startswith("active")})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(self.rows)}


def thermo(args, grid):
    from paper_2409_07232_b200 import synth
    return synth.thermo_host(args.ni, args.nk, args.nj, args.cf, CONFIG["seed"], grid)


def make_ctx(nkr, device=0):
    import paper_2409_07232_b200 as fsbm
    grid = fsbm.make_mass_grid(nkr, 3.35e-14, fsbm.equal_range_ratio(nkr))
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1.0, 1.5, 0.05))
    return fsbm.CoalContext(grid, tabs, device), grid, tabs


# ---------------------------------------------------------------------------------------
# CPU reference leg (oracle/_ref = the reference's own fissioned_step)
# ---------------------------------------------------------------------------------------
def reference_sample(args, grid, tabs, rows, B_slab=None, T=None, P=None):
    """Times the reference fissioned_step on the first `rows` i-rows of the workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    R = pyoracle.Reference()
    per_i = args.nk * args.nj
    npts = rows * per_i
    if B_slab is None:
        O = pyoracle.Oracle()
        mask = ((T[:npts] > 193.15) & (T[:npts] > 223.15)).astype(np.uint8)
        B_slab = O.thunderstorm_block(grid.x, CONFIG["seed"], 0, npts, mask)
    B = np.ascontiguousarray(B_slab)
    cores = os.cpu_count() or 1
    st, cnt, tim, err = R.fissioned_step(rows, args.nk, args.nj, grid.nkr(),
                                         tabs.t750.reshape(-1).copy(), tabs.t500.reshape(-1).copy(),
                                         np.ascontiguousarray(T[:npts]),
                                         np.ascontiguousarray(P[:npts]), B, CONFIG["dt"],
                                         CONFIG["substeps"], mode=1, collapse=3, threads=cores,
                                         kernel_strategy=1, scratch_strategy=1,
                                         ratio=grid.ratio)
    if st != 0:
        raise RuntimeError(f"reference fissioned_step failed: {R.last_error()}")
    return int(cnt[1]) / tim[0], cores, int(cnt[1]), tim[0]


def pick_rows(args, grid, tabs, T, P, gen, target_s):
    """Calibrate on one i-row, then size the sample for ~target_s of wall time."""
    rate, cores, n, t = reference_sample(args, grid, tabs, 1, gen(1), T, P)
    rows = int(max(1, min(args.ni, 120, target_s * rate / (args.nk * args.nj))))
    return rows, rate


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_2409_07232_b200 as fsbm
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    grid = fsbm.make_mass_grid(args.nkr, 3.35e-14, fsbm.equal_range_ratio(args.nkr))
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1.0, 1.5, 0.05))
    T, P, _ = thermo(args, grid)
    O = pyoracle.Oracle()
    per_i = args.nk * args.nj

    def gen(rows):
        n = rows * per_i
        m = ((T[:n] > 193.15) & (T[:n] > 223.15)).astype(np.uint8)
        return O.thunderstorm_block(grid.x, CONFIG["seed"], 0, n, m)

    target = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rows, _ = pick_rows(args, grid, tabs, T, P, gen, target)
    B = gen(rows)
    rates, cores = [], os.cpu_count() or 1
    for s in range(args.warmup + args.steps):
        r, cores, n, t = reference_sample(args, grid, tabs, rows, B.copy(), T, P)
        if s >= args.warmup:
            rates.append(r)
    value = statistics.median(rates)
    sample = (f"{rows} of {args.ni} i-rows ({rows * per_i} points) of the C2 thunderstorm grid "
              f"per step; reference fissioned_step collapse-3 arena on_demand, {cores} threads, "
              f"timed by its PhaseTimings.coal_s")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * (args.ni * per_i) / value, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_label(args):
    """BASELINE.json configs: C2 (33 bins) is the headline; C3/C4 (66/132 bins) share its
    grid; C5 (264 bins, 850x600x50 over 8 GPUs) is run as one GPU's patch."""
    if (args.ni, args.nj, args.nk) == (425, 300, 50):
        return {33: "C2", 66: "C3", 132: "C4"}.get(args.nkr, "C2-grid")
    if args.nkr == 264 and (args.nj, args.nk) == (600, 50):
        return "C5 per-GPU patch"
    return "custom"


def config_block(args, world):
    scale = getattr(args, "scaling", "weak")
    ni_g = args.ni * world if scale == "weak" else args.ni
    return {"workload": f"{config_label(args)} CONUS-12km {args.ni}x{args.nj}x{args.nk} (i x j x k) per GPU"
                        f"{' (weak: N stacked C2 slabs)' if scale == 'weak' and world > 1 else ''}, "
                        f"{args.nkr} bins, thunderstorm all-category input, cf {args.cf}, "
                        f"dt 1 s, 1 substep",
            "grid": [args.ni, args.nj, args.nk], "nkr": args.nkr, "pairs": 20,
            "global_points": ni_g * args.nj * args.nk,
            "parallelism": f"i-slab shards x{world} (no halo; NCCL diagnostics only)",
            "numerics": args.numerics,
            "l2": "state (6 x 1.68 GB) >> 126 MB L2, and restored before every step"}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2409_07232_b200 as fsbm
    from paper_2409_07232_b200 import _lib, shard, synth

    world, rank, local = dist_env()
    # FSBM_BENCH_ONE_GPU=1 (plumbing check only): every rank on cuda:0 over gloo, so the
    # N>1 sharding / reduction path can be exercised on a one-GPU box; never a bench number
    if os.environ.get("FSBM_BENCH_ONE_GPU") == "1":
        local = 0
    if world > 1:
        if os.environ.get("FSBM_BENCH_ONE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    lib = _lib.load()

    ctx, grid, tabs = make_ctx(args.nkr, local)
    nkr = args.nkr
    ni_global = args.ni * world if args.scaling == "weak" else args.ni
    T, P, _ = synth.thermo_host(ni_global, args.nk, args.nj, args.cf, CONFIG["seed"], grid)
    i0, i1 = shard.slab(ni_global, world, rank)
    state, mask = synth.thunderstorm_device(ctx, ni_global, args.nk, args.nj, args.cf,
                                            CONFIG["seed"], device=dev, i_slab=(i0, i1),
                                            thermo=(T, P, None))
    pristine = [b.clone() for b in state.bins]
    npts_local = (i1 - i0) * args.nk * args.nj
    plan = fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", args.numerics)
    stream = torch.cuda.current_stream(dev)
    cnt = fsbm.WorkCounters()
    sctx = fsbm.StepContext(ctx, fsbm.CoalConfig(CONFIG["dt"], CONFIG["substeps"]), cnt,
                            stream=stream.cuda_stream)

    def restore():
        for b, p in zip(state.bins, pristine):
            b.copy_(p, non_blocking=True)

    xs = torch.from_numpy(grid.x).to(dev)

    def mass():
        return torch.stack([(b.view(-1, nkr) * xs).sum() for b in state.bins]).sum()

    # ---- warm-up ----
    for _ in range(args.warmup):
        restore()
        fsbm.fissioned_step(state, mask, sctx, plan)
    torch.cuda.synchronize()
    # ---- timed ----
    e_beg = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_end = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kern_ms, launches = [], 0
    cnt.triples = cnt.points = cnt.kernel_evals = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for s in range(args.steps):
            restore()
            e_beg[s].record(stream)
            fsbm.fissioned_step(state, mask, sctx, plan)
            e_end[s].record(stream)
            km, nl = C.c_float(), C.c_int()
            lib.fsbm_ctx_last_timing(ctx.handle, C.byref(km), C.byref(nl))
            kern_ms.append(km.value)
            launches += nl.value
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
    step_ms = sum(a.elapsed_time(b) for a, b in zip(e_beg, e_end)) / args.steps
    kernel_ms = sum(kern_ms) / len(kern_ms)
    # diagnostics (the only collective: one NCCL all-reduce of a few scalars)
    restore()
    m0 = mass()
    fsbm.fissioned_step(state, mask, fsbm.StepContext(ctx, sctx.coal, None, stream=stream.cuda_stream), plan)
    m1 = mass()
    diag = shard.reduce_diagnostics(
        shard.StepDiagnostics(cnt.triples // args.steps, cnt.points // args.steps,
                              cnt.kernel_evals // args.steps, m0.item(), m1.item()), dist, dev)
    tmax = torch.tensor([step_ms, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)  # device time: max over ranks
    step_ms_max, kernel_ms_max = tmax.tolist()
    points, triples, m0g, m1g = float(diag.points), float(diag.triples), diag.mass_before, diag.mass_after
    value = points / (step_ms_max * 1e-3)

    # ---- roofline (FP64 pipe; algorithmic flops) ----
    peak = C.c_double()
    _lib.check(lib.fsbm_probe_fp64_peak(local, C.byref(peak)))
    local_triples = cnt.triples / args.steps
    achieved = FLOP_PER_TRIPLE * local_triples / (kernel_ms * 1e-3) / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
            "frac": achieved / peak.value, "traffic": None,
            "peak_source": "measured live: fsbm_probe_fp64_peak DFMA-chain microbenchmark "
                           "(MEASURED_PEAKS.json has no FP64 entry)",
            "kernel": ctx.fast_kernel() if args.numerics == "fast" else "coal_exact",
            "flop_per_update": FLOP_PER_TRIPLE * local_triples / max(1.0, cnt.points / args.steps),
            "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / step_ms,
            "hbm_bytes_per_update": 96 * nkr + 16}
    hbm_gbs = (96 * nkr + 16) * (cnt.points / args.steps) / (kernel_ms * 1e-3) / 1e9
    roof["hbm_algorithmic_gbs"] = hbm_gbs
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        roof["hbm_frac_of_measured"] = hbm_gbs / peaks["hbm_gbs"]
    except Exception:
        pass
    try:  # DRAM bytes of the coal kernel from the committed ncu --set full capture, per launch
        tr = json.load(open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")))["by_nkr"].get(str(nkr))
        if tr:
            roof["traffic"] = tr["bytes_per_update"] * (cnt.points / args.steps)
            roof["traffic_source"] = tr["source"]
    except Exception:
        pass

    # ---- e2e through the host C ABI ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, state, pristine, T, P, i0, i1, plan, world)

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        try:
            per_i = args.nk * args.nj

            def gen(rows):
                return torch.stack([p.view(-1, nkr)[: rows * per_i] for p in pristine]).cpu().numpy()

            rows, _ = pick_rows(args, grid, tabs, T, P, gen, args.cpu_seconds)
            rate, cores, n, t = reference_sample(args, grid, tabs, rows, gen(rows), T, P)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"{rows} of {args.ni} i-rows ({n} points, same input bytes) of this "
                             f"workload; reference fissioned_step collapse-3 arena on_demand with "
                             f"{cores} threads; {t:.2f} s by PhaseTimings.coal_s"}
        except Exception as ex:  # the reference .so may be absent on a stripped tree
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (SURVEY 8(d) thunderstorm builder; golovin tables)",
                "config": config_block(args, world),
                "e2e": e2e, "gpu_launches": launches * world,
                "roofline": roof, "cpu_baseline": cpu,
                "clocks": clk.summary(),
                "diagnostics": {"updates_per_step": points, "triples_per_step": triples,
                                "mass_before": m0g, "mass_after": m1g,
                                "mass_rel_drift": abs(m1g - m0g) / m0g, "wall_s_timed": wall}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, ctx, state, pristine, T, P, i0, i1, plan, world):
    """Same metric through fsbm_step_grid_host (host buffers, H2D + step + D2H timed)."""
    import torch
    import torch.distributed as dist

    import paper_2409_07232_b200 as fsbm

    per_i = args.nk * args.nj
    n = (i1 - i0) * per_i
    host_bins = [torch.empty(p.numel(), dtype=torch.float64, pin_memory=True) for p in pristine]
    hT = torch.from_numpy(np.ascontiguousarray(T[i0 * per_i:i1 * per_i])).pin_memory()
    hP = torch.from_numpy(np.ascontiguousarray(P[i0 * per_i:i1 * per_i])).pin_memory()
    hstate = fsbm.GridState(state.ranges, state.grid, hT.numpy(), hP.numpy(),
                            [h.numpy() for h in host_bins])
    cnt = fsbm.WorkCounters()
    sctx = fsbm.StepContext(ctx, fsbm.CoalConfig(CONFIG["dt"], CONFIG["substeps"]), cnt)
    times = []
    for s in range(1 + args.e2e_steps):
        for h, p in zip(host_bins, pristine):  # restore input (not timed)
            h.copy_(p)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        fsbm.fissioned_step(hstate, None, sctx, plan)
        dt = time.perf_counter() - t0
        if s > 0:
            times.append(dt)
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=state.bins[0].device)
    pts = torch.tensor([float(cnt.points) / (1 + args.e2e_steps)], dtype=torch.float64,
                       device=state.bins[0].device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(pts, op=dist.ReduceOp.SUM)
    h2d = 6 * n * args.nkr * 8 + 2 * n * 8
    d2h = 6 * n * args.nkr * 8
    return {"value": pts.item() / t.item(), "unit": UNIT, "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "s_per_step": t.item(),
            "path": "fsbm_step_grid_host (pinned host GridState arrays)"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
