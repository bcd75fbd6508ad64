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
no halo), stepped through the library's device group (fsbm_group_step_device, one group
per rank) whose only collective is its own NCCL all-reduce of the end-of-step counters
and diagnostics.  The thunderstorm
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
           on-demand, all host threads) on a bounded sample of the same bytes
parity     that sample's reference output against the GPU output of the timed
           configuration at the same points (SURVEY 8(c) bar), counters exact
exact      FSBM_NUMERICS_EXACT (bitwise coal_step) throughput at C2 + bitwise check
configs    C3 / C4 (66 / 132 bins, C2 grid) and one GPU's C5 patch (264 bins), each
           with value, roofline, cpu_baseline and parity (N=1 only); C2-cf03 (the
           SURVEY 8(d) imbalance test: a scattered cloud-fraction-0.3 mask); C2-dense (every bin
           non-zero: no zero-product skips); C2-bott (the C2 workload through Bott's flux
           method, FSBM_NUMERICS_BOTT, checked against the C port oracle/bott_oracle.c)

--impl reference runs the reference alone (rank 0): oracle/_ref's fissioned_step on a
bounded sample of the same workload; its inputs come from the checkers under oracle/
(make_synthetic_case's T/P recipe, the thunderstorm builder), never from this package.
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
X1 = 3.35e-14
RTOL, ATOL_FRAC = 1e-12, 1e-15  # SURVEY 8(c) per-bin bar
# The dense input (every bin non-zero) is stiff at dt = 1 s with these tables (a top-bin
# loss rate of ~x_top * N ~ 360/s), so it steps dt = 1 ms: the same work per update.
DENSE_DT = 1e-3


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
    ap.add_argument("--input", default="thunderstorm", choices=["thunderstorm", "dense"],
                    help="dense: every bin of every category non-zero (no zero-product skips)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip cpu_baseline and parity")
    ap.add_argument("--no-exact", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--configs", default="C3,C4,C5,C2-cf03,C2-dense,C2-bott")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--cfg-cpu-seconds", type=float, default=5.0)
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


# ---------------------------------------------------------------------------------------
# the reference's fissioned_step on a bounded sample (checkers under oracle/ only)
# ---------------------------------------------------------------------------------------
def checkers():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    return pyoracle


class RefCase:
    """Tables from the reference itself (build_tables with golovin/1/1.5/0.05)."""

    def __init__(self, nkr):
        po = checkers()
        self.R, self.O = po.Reference(), po.Oracle()
        self.nkr = nkr
        self.ratio = po.equal_range_ratio(nkr)
        self.x = self.R.mass_grid(nkr, X1, self.ratio)
        self.t750, self.t500 = self.R.build_tables(nkr, X1, self.ratio, family=1, coeff=1.0,
                                                   level_scale=1.5, pair_scale_step=0.05)

    def run(self, ri, nk, njs, T, P, B):
        """fissioned_step (collapse-3 arena, on_demand, all host threads) on a (ri, nk, njs)
        grid, B (6, n, nkr) updated in place.  Returns (points/s, counters, coal_s, cores)."""
        cores = os.cpu_count() or 1
        st, cnt, tim, err = self.R.fissioned_step(ri, nk, njs, self.nkr, self.t750, self.t500,
                                                  np.ascontiguousarray(T), np.ascontiguousarray(P),
                                                  B, CONFIG["dt"], CONFIG["substeps"], mode=1,
                                                  collapse=3, threads=cores, kernel_strategy=1,
                                                  scratch_strategy=1, x1=X1, ratio=self.ratio)
        if st != 0:
            raise RuntimeError(f"reference fissioned_step failed: {self.R.last_error()}")
        return int(cnt[1]) / tim[0], [int(v) for v in cnt], float(tim[0]), cores


class BottCase:
    """CPU port of Bott's flux method (oracle/bott_oracle.c; the reference has no such scheme,
    SPEC.md:226), same tables as RefCase, all host threads."""

    def __init__(self, nkr):
        po = checkers()
        self.O = po.Oracle()
        self.nkr = nkr
        self.ratio = po.equal_range_ratio(nkr)
        self.x = self.O.mass_grid(nkr, X1, self.ratio)
        self.t750, self.t500 = self.O.build_tables(self.x, npairs=20, family=1, coeff=1.0,
                                                   level_scale=1.5, pair_scale_step=0.05)
        self.abd = self.O.default_registry()
        self.lo = self.O.gain_table(self.x, self.ratio)[0]
        self.cour = self.O.bott_courant(self.x, self.lo)

    def run(self, ri, nk, njs, T, P, B):
        cores = os.cpu_count() or 1
        mask, _ = self.O.fission_predicates(np.ascontiguousarray(T))
        t0 = time.perf_counter()
        st, cnt = self.O.bott_step_grid(self.x, self.abd, self.t750, self.t500, self.lo, self.cour,
                                        mask, np.ascontiguousarray(P), B, CONFIG["dt"],
                                        CONFIG["substeps"], 1, cores)
        secs = time.perf_counter() - t0
        if st != 0:
            raise RuntimeError("oracle bott_step_grid failed")
        return int(cnt[1]) / secs, [int(v) for v in cnt], secs, cores


def sample_index(ni, nk, nj, ri, njs):
    """Flat point indices of the sub-box i < ri, all k, j < njs, in the reference layout
    of a (ri, nk, njs) grid."""
    i = np.arange(ri)[:, None, None]
    k = np.arange(nk)[None, :, None]
    j = np.arange(njs)[None, None, :]
    return ((i * nk + k) * nj + j).reshape(-1)


def size_sample(ni, nk, nj, points):
    """(ri, njs): whole i-rows when the budget allows, else one row's first j-columns."""
    per_i = nk * nj
    if points >= per_i:
        return int(min(ni, points // per_i)), nj
    return 1, int(max(1, min(nj, points // nk)))


def run_reference_arm(args):
    """Reference arm: rank 0 only; never imports paper_2409_07232_b200."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    ref = RefCase(args.nkr)
    ni = args.ni * world if args.scaling == "weak" else args.ni
    nk, nj = args.nk, args.nj
    T, P, _ = ref.O.synthetic_case(ni, nk, nj, args.cf, CONFIG["seed"], args.nkr, X1, ref.ratio,
                                   spectra=False)

    def inputs(ri, njs):
        idx = sample_index(ni, nk, nj, ri, njs)
        Ts, Ps = T[idx], P[idx]
        mask, _ = ref.O.fission_predicates(Ts)
        if njs == nj:  # whole i-rows: the grid's first points, contiguous
            return Ts, Ps, ref.O.thunderstorm_block(ref.x, CONFIG["seed"], 0, idx.size, mask)
        B = np.zeros((6, idx.size, args.nkr))
        for q in np.nonzero(mask)[0]:  # thunderstorm spectra keyed by the GLOBAL point index
            B[:, q] = ref.O.thunderstorm_point(ref.x, CONFIG["seed"], int(idx[q]))
        return Ts, Ps, B

    if args.input == "dense":
        raise SystemExit("--impl reference --input dense: not a reference workload")
    cal = size_sample(ni, nk, nj, 2000)
    Ts, Ps, B = inputs(*cal)
    rate0, _, _, _ = ref.run(cal[0], nk, cal[1], Ts, Ps, B)
    target_s = max(2.0, min(20.0, 100.0 / max(1, args.steps + args.warmup)))
    ri, njs = size_sample(ni, nk, nj, int(rate0 * target_s))
    Ts, Ps, B = inputs(ri, njs)
    rates, secs, cores = [], [], 1
    for s in range(args.warmup + args.steps):
        r, _, t, cores = ref.run(ri, nk, njs, Ts, Ps, B.copy())
        if s >= args.warmup:
            rates.append(r)
            secs.append(t)
    value = statistics.median(rates)
    npts = ri * nk * njs
    sample = (f"{ri} i-row(s) x {nk} k x {njs} j ({npts} points) of the {ni}x{nj}x{nk} "
              f"{args.nkr}-bin thunderstorm grid per step (the grid's first points); reference "
              f"fissioned_step collapse-3 arena on_demand, {cores} threads, timed by its "
              f"PhaseTimings.coal_s; ms_per_step is that sample's measured step time")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(secs), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "inputs": "T/P: oracle restatement of make_synthetic_case (bitwise equal to the "
                      "reference's, tests/test_oracle.py); tables: reference build_tables; "
                      "spectra: oracle thunderstorm builder"}
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
    inp = getattr(args, "input", "thunderstorm")
    return {"workload": f"{config_label(args)} CONUS-12km {args.ni}x{args.nj}x{args.nk} (i x j x k) per GPU"
                        f"{' (weak: N stacked C2 slabs)' if scale == 'weak' and world > 1 else ''}, "
                        f"{args.nkr} bins, {inp} all-category input, cf {args.cf}, "
                        f"dt {DENSE_DT if inp == 'dense' else 1} s, 1 substep",
            "grid": [args.ni, args.nj, args.nk], "nkr": args.nkr, "pairs": 20,
            "global_points": ni_g * args.nj * args.nk,
            "parallelism": f"i-slab shards x{world} (no halo; NCCL diagnostics only)",
            "numerics": args.numerics,
            "l2": "state (6 x 1.68 GB) >> 126 MB L2, and restored before every step"}


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def make_ctx(nkr, device=0):
    import paper_2409_07232_b200 as fsbm
    grid = fsbm.make_mass_grid(nkr, X1, fsbm.equal_range_ratio(nkr))
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1.0, 1.5, 0.05))
    return fsbm.CoalContext(grid, tabs, device), grid, tabs


def fp64_peak(dev_index):
    import ctypes as C
    from paper_2409_07232_b200 import _lib
    peak = C.c_double()
    _lib.check(_lib.load().fsbm_probe_fp64_peak(dev_index, C.byref(peak)))
    return peak.value


def ncu_traffic(nkr, points, tag=None):
    """DRAM bytes of the coal kernel per launch from a committed ncu --set full capture."""
    for name in ("r02_ncu_traffic.json", "r01_ncu_traffic.json"):  # newest capture first
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", name)))["by_nkr"]
        except Exception:
            continue
        e = tr.get(tag or str(nkr))
        if e:
            return e["bytes_per_update"] * points, e["source"]
    return None, None


def roofline(nkr, triples, points, kernel_ms, peak, kernel, tag=None):
    achieved = FLOP_PER_TRIPLE * triples / (kernel_ms * 1e-3) / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": None,
            "peak_source": "measured live: fsbm_probe_fp64_peak DFMA-chain microbenchmark "
                           "(MEASURED_PEAKS.json has no FP64 entry)",
            "kernel": kernel, "flop_per_update": FLOP_PER_TRIPLE * triples / max(1.0, points),
            "kernel_ms": kernel_ms, "hbm_bytes_per_update": 96 * nkr + 16}
    hbm_gbs = (96 * nkr + 16) * points / (kernel_ms * 1e-3) / 1e9
    roof["hbm_algorithmic_gbs"] = hbm_gbs
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        roof["hbm_frac_of_measured"] = hbm_gbs / peaks["hbm_gbs"]
    except Exception:
        pass
    tr, src = ncu_traffic(nkr, points, tag)
    if tr is not None:
        roof["traffic"] = tr
        roof["traffic_source"] = src
    return roof


def gather(bins, idx_t, nkr):
    """(6, n, nkr) device tensor of the given points of a device GridState."""
    import torch
    return torch.stack([b.view(-1, nkr).index_select(0, idx_t) for b in bins])


def parity_block(got, ref_out, B_in, x, cnt_gpu, cnt_ref, exact_equal, sample):
    """SURVEY 8(c) bar on device: per bin |gpu-ref| <= 1e-12|ref| + 1e-15*sum_k ref_c;
    per-point mass |sum n.x after - before| <= 1e-12 before; number non-increasing."""
    import torch
    dev = got.device
    xs = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    bad, max_rel, tol_frac = 0, 0.0, 0.0
    m_in = m_out = n_in = n_out = None
    for c in range(6):
        r = torch.from_numpy(np.ascontiguousarray(ref_out[c])).to(dev)
        g = got[c]
        d = (g - r).abs()
        tol = RTOL * r.abs() + ATOL_FRAC * r.abs().sum(-1, keepdim=True)
        bad += int((d > tol).sum())
        nz = r != 0
        if bool(nz.any()):
            max_rel = max(max_rel, float((d[nz] / r[nz].abs()).max()))
        tol_frac = max(tol_frac, float((d / tol.clamp_min(1e-300)).max()))
        bi = torch.from_numpy(np.ascontiguousarray(B_in[c])).to(dev)
        mi, mo = (bi * xs).sum(-1), (g * xs).sum(-1)
        m_in = mi if m_in is None else m_in + mi
        m_out = mo if m_out is None else m_out + mo
        n_in = bi.sum(-1) if n_in is None else n_in + bi.sum(-1)
        n_out = g.sum(-1) if n_out is None else n_out + g.sum(-1)
        del r, d, tol, bi
    pos = m_in > 0
    mass_rel = float(((m_out - m_in).abs()[pos] / m_in[pos]).max()) if bool(pos.any()) else 0.0
    return {"sample": sample, "points": int(got.shape[1]), "bins_compared": int(got.numel()),
            "bins_out_of_tol": bad, "max_rel": max_rel, "max_err_over_tol": tol_frac,
            "tolerance": "per bin |gpu-ref| <= 1e-12|ref| + 1e-15*sum_k ref_c[k] (SURVEY 8(c))",
            "counters_gpu": cnt_gpu, "counters_ref": cnt_ref, "counters_equal": cnt_gpu == cnt_ref,
            "point_mass_max_rel_drift": mass_rel, "mass_ok": mass_rel <= 1e-12,
            "number_non_increasing": bool((n_out <= n_in * (1 + 1e-15)).all()),
            "exact_bitwise_vs_reference": exact_equal,
            "green": bad == 0 and cnt_gpu == cnt_ref and mass_rel <= 1e-12
            and exact_equal is not False}


def sample_parity(fsbm, ctx, grid, ref, dims, T, P, pristine, out_bins, seconds, dev):
    """cpu_baseline + parity on one bounded sample.  pristine/out_bins: the config's input
    and its GPU output (full timed configuration) as lists of 6 flat device tensors."""
    import torch
    ni, nk, nj = dims
    nkr = grid.nkr()
    cal = size_sample(ni, nk, nj, 2000)
    idx = sample_index(ni, nk, nj, *cal)
    idx_t = torch.from_numpy(idx).to(dev)
    B = gather(pristine, idx_t, nkr).cpu().numpy()
    rate0, _, _, _ = ref.run(cal[0], nk, cal[1], T[idx], P[idx], B)
    ri, njs = size_sample(ni, nk, nj, int(rate0 * seconds))
    idx = sample_index(ni, nk, nj, ri, njs)
    idx_t = torch.from_numpy(idx).to(dev)
    B_in = gather(pristine, idx_t, nkr).cpu().numpy()
    Ts, Ps = T[idx], P[idx]
    ref_out = B_in.copy()
    rate, cnt_ref, secs, cores = ref.run(ri, nk, njs, Ts, Ps, ref_out)
    got = gather(out_bins, idx_t, nkr)
    # counters of exactly the sample through the product (same bytes, sub-grid), and the
    # EXACT kernel's bitwise check on it
    sub = fsbm.Ranges(1, ri, 1, nk, 1, njs)
    Td, Pd = torch.from_numpy(Ts).to(dev), torch.from_numpy(Ps).to(dev)
    cnt = fsbm.WorkCounters()
    st = fsbm.GridState(sub, grid, Td, Pd, [torch.from_numpy(B_in[c].reshape(-1)).to(dev)
                                            for c in range(6)])
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, counters=cnt),
                        fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", "fast"))
    del st
    st = fsbm.GridState(sub, grid, Td, Pd, [torch.from_numpy(B_in[c].reshape(-1)).to(dev)
                                            for c in range(6)])
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx),
                        fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", "exact"))
    ex = torch.stack([b.view(-1, nkr) for b in st.bins]).cpu().numpy()
    exact_equal = bool(np.array_equal(ex, ref_out))
    del st, ex
    desc = f"{ri} i-row(s) x {nk} k x {njs} j ({idx.size} points): the grid's first points"
    par = parity_block(got, ref_out, B_in, grid.x,
                       [cnt.triples, cnt.points, cnt.kernel_evals], cnt_ref, exact_equal, desc)
    cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
           "sample": f"{desc} of this workload, same input bytes; reference fissioned_step "
                     f"collapse-3 arena on_demand with {cores} threads; {secs:.2f} s by "
                     f"PhaseTimings.coal_s"}
    return cpu, par


def bott_sample_parity(fsbm, ctx, grid, dims, T, P, pristine, out_bins, seconds, dev):
    """cpu_baseline (the C port of Bott's scheme on all host threads, kind "port") and parity
    of the GPU's Bott output against it on one bounded sample of the same bytes."""
    import torch
    ni, nk, nj = dims
    nkr = grid.nkr()
    bc = BottCase(nkr)
    cal = size_sample(ni, nk, nj, 2000)
    idx = sample_index(ni, nk, nj, *cal)
    B = gather(pristine, torch.from_numpy(idx).to(dev), nkr).cpu().numpy()
    rate0, _, _, _ = bc.run(cal[0], nk, cal[1], T[idx], P[idx], B)
    ri, njs = size_sample(ni, nk, nj, int(rate0 * seconds))
    idx = sample_index(ni, nk, nj, ri, njs)
    idx_t = torch.from_numpy(idx).to(dev)
    B_in = gather(pristine, idx_t, nkr).cpu().numpy()
    ref_out = np.ascontiguousarray(B_in.copy())
    rate, cnt_ref, secs, cores = bc.run(ri, nk, njs, T[idx], P[idx], ref_out)
    got = gather(out_bins, idx_t, nkr)
    sub = fsbm.Ranges(1, ri, 1, nk, 1, njs)
    cnt = fsbm.WorkCounters()
    st = fsbm.GridState(sub, grid, torch.from_numpy(T[idx]).to(dev), torch.from_numpy(P[idx]).to(dev),
                        [torch.from_numpy(B_in[c].reshape(-1)).to(dev) for c in range(6)])
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, counters=cnt),
                        fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", "bott"))
    del st
    desc = f"{ri} i-row(s) x {nk} k x {njs} j ({idx.size} points): the grid's first points"
    par = parity_block(got, ref_out, B_in, grid.x, [cnt.triples, cnt.points, cnt.kernel_evals],
                       cnt_ref, None, desc)
    par["checker"] = "oracle/bott_oracle.c (KAT-pinned restatement of Bott 1998; no reference scheme)"
    cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
           "sample": f"{desc} of this workload, same input bytes; oracle bott_step_grid with {cores} "
                     f"threads; {secs:.2f} s wall"}
    return cpu, par


def regen(lib, ctx, state, mask, offset, seed, dense, stream):
    """Re-generate a config's input in place (outside the timed events)."""
    import ctypes as C

    from paper_2409_07232_b200 import _lib
    ptrs = (C.c_void_p * 6)(*[b.data_ptr() for b in state.bins])
    _lib.check(lib.fsbm_synth_thunderstorm_device(ctx.handle, state.bins[0].numel() // ctx.nkr,
                                                  offset, mask.call_coal.data_ptr(), seed, ptrs,
                                                  stream))
    if dense:
        densify(state, mask, ctx.grid)


def densify(state, mask, grid):
    """Dense secondary input: every bin of every category non-zero at mask-true points
    (the thunderstorm spectra underflow to exact zeros in their upper bins, which the
    kernels legitimately skip; this input has nothing to skip).  1e-3 per bin is added;
    the step uses DENSE_DT."""
    import torch
    on = mask.call_coal.bool()
    for b in state.bins:
        v = b.view(-1, grid.nkr())
        v[on] = v[on] + 1e-3


def timed_steps(fsbm, lib, ctx, state, mask, plan, steps, prep, stream, dt=CONFIG["dt"]):
    """steps x (prep outside events -> events around fissioned_step); returns
    (mean step ms, mean coal-kernel ms, launches, counters)."""
    import ctypes as C

    import torch
    cnt = fsbm.WorkCounters()
    sctx = fsbm.StepContext(ctx, fsbm.CoalConfig(dt, CONFIG["substeps"]), cnt,
                            stream=stream.cuda_stream)
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    km, launches = [], 0
    for s in range(steps):
        prep()
        e0[s].record(stream)
        fsbm.fissioned_step(state, mask, sctx, plan)
        e1[s].record(stream)
        k, n = C.c_float(), C.c_int()
        lib.fsbm_ctx_last_timing(ctx.handle, C.byref(k), C.byref(n))
        km.append(k.value)
        launches += n.value
    torch.cuda.synchronize()
    return (sum(a.elapsed_time(b) for a, b in zip(e0, e1)) / steps, sum(km) / steps, launches,
            cnt)


def run_config(args, label, nkr, dims, dev, peak, steps=3, dense=False, offset_rows=0,
               numerics="fast", cf=None):
    """One secondary BASELINE config on this GPU: value, roofline, cpu_baseline, parity.
    numerics="bott": the same workload through Bott's flux method."""
    import torch

    import paper_2409_07232_b200 as fsbm
    from paper_2409_07232_b200 import _lib, synth
    lib = _lib.load()
    ni, nk, nj = dims
    ctx, grid, tabs = make_ctx(nkr, dev.index or 0)
    ni_g = ni if not offset_rows else offset_rows
    cf = args.cf if cf is None else cf
    T, P, _ = synth.thermo_host(ni_g, nk, nj, cf, CONFIG["seed"], grid)
    T, P = T[:ni * nk * nj].copy(), P[:ni * nk * nj].copy()
    state, mask = synth.thunderstorm_device(ctx, ni, nk, nj, cf, CONFIG["seed"], device=dev,
                                            thermo=(T, P, None))
    stream = torch.cuda.current_stream(dev)
    plan = fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", numerics)

    def prep():
        regen(lib, ctx, state, mask, 0, CONFIG["seed"], dense, stream.cuda_stream)

    dt = DENSE_DT if dense else CONFIG["dt"]
    timed_steps(fsbm, lib, ctx, state, mask, plan, 1, prep, stream, dt)  # warm-up
    step_ms, kern_ms, _, cnt = timed_steps(fsbm, lib, ctx, state, mask, plan, steps, prep, stream,
                                           dt)
    points, triples = cnt.points / steps, cnt.triples / steps
    kname = ctx.fast_kernel() if numerics == "fast" else f"coal_{numerics}"
    out = {"workload": f"{label}: {ni}x{nj}x{nk} (i x j x k), {nkr} bins, "
                       f"{'dense' if dense else 'thunderstorm'} all-category input, cf {cf}, "
                       f"dt {dt:g} s" + (", Bott (1998) flux method" if numerics == "bott" else ""),
           "value": points / (step_ms * 1e-3), "unit": UNIT, "ms_per_step": step_ms,
           "steps": steps, "updates_per_step": points,
           "roofline": roofline(nkr, triples, points, kern_ms, peak, kname,
                                tag=f"{nkr}-dense" if dense else (f"{nkr}-{numerics}" if numerics != "fast" else None))}
    out["roofline"]["kernel_share_of_step"] = kern_ms / step_ms
    if numerics == "bott":
        out["roofline"]["note"] = ("SURVEY 8(d)'s 12 FLOP per visited triple, the same work unit as "
                                   "Kovetz-Olund; Bott's sweep is sequential per point (Gauss-Seidel) "
                                   "and adds log/exp per non-zero triple: latency-bound, one point per thread")
    if not args.no_cpu and not dense and numerics == "bott":
        prep()
        pristine = [b.clone() for b in state.bins]
        fsbm.fissioned_step(state, mask, fsbm.StepContext(ctx, stream=stream.cuda_stream), plan)
        out["cpu_baseline"], out["parity"] = bott_sample_parity(fsbm, ctx, grid, dims, T, P, pristine,
                                                                state.bins, args.cfg_cpu_seconds, dev)
        del pristine
    elif not args.no_cpu and not dense:
        prep()
        pristine = [b.clone() for b in state.bins]
        fsbm.fissioned_step(state, mask, fsbm.StepContext(ctx, stream=stream.cuda_stream), plan)
        try:
            ref = RefCase(nkr)
            cpu, par = sample_parity(fsbm, ctx, grid, ref, dims, T, P, pristine, state.bins,
                                     args.cfg_cpu_seconds, dev)
            out["cpu_baseline"], out["parity"] = cpu, par
        except Exception as ex:  # the reference .so may be absent on a stripped tree
            out["cpu_baseline"] = {"value": None, "sample": f"unavailable: {ex}"}
        del pristine
    del state, mask, ctx
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


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
    dense = args.input == "dense"
    ni_global = args.ni * world if args.scaling == "weak" else args.ni
    T, P, _ = synth.thermo_host(ni_global, args.nk, args.nj, args.cf, CONFIG["seed"], grid)
    i0, i1 = shard.slab(ni_global, world, rank)
    state, mask = synth.thunderstorm_device(ctx, ni_global, args.nk, args.nj, args.cf,
                                            CONFIG["seed"], device=dev, i_slab=(i0, i1),
                                            thermo=(T, P, None))
    if dense:
        densify(state, mask, grid)
    pristine = [b.clone() for b in state.bins]
    plan = fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", args.numerics)
    stream = torch.cuda.current_stream(dev)
    cnt = fsbm.WorkCounters()
    step_dt = DENSE_DT if dense else CONFIG["dt"]
    sctx = fsbm.StepContext(ctx, fsbm.CoalConfig(step_dt, CONFIG["substeps"]), cnt,
                            stream=stream.cuda_stream)

    def restore():
        for b, p in zip(state.bins, pristine):
            b.copy_(p, non_blocking=True)

    xs = torch.from_numpy(grid.x).to(dev)

    def mass():
        return torch.stack([(b.view(-1, nkr) * xs).sum() for b in state.bins]).sum()

    # N > 1: the step goes through the library's device group (include/fsbm_coal.h,
    # fsbm_group_*): one group per rank, counters / first failing point / diagnostics
    # reduced by the library's own NCCL all-reduce; the NCCL id travels
    # over torch.distributed.  (FSBM_BENCH_ONE_GPU plumbing runs keep the per-rank path.)
    group = None
    # FSBM_BENCH_GROUP=1 takes the group path at N=1 too (a one-rank group, no NCCL): a
    # plumbing check of the N>1 code on a one-GPU box
    if (world > 1 and os.environ.get("FSBM_BENCH_ONE_GPU") != "1") or os.environ.get("FSBM_BENCH_GROUP") == "1":
        from paper_2409_07232_b200 import group as fgroup
        obj = [fgroup.nccl_unique_id() if rank == 0 and world > 1 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        group = fgroup.DeviceGroup(grid, tabs, [local], rank, world, obj[0])
        gctx = group.ctx_handle(0)

    def one_step(counters=cnt, diagnostics=False):
        if group is None:
            fsbm.fissioned_step(state, mask, fsbm.StepContext(ctx, sctx.coal, counters,
                                                              stream=stream.cuda_stream), plan)
            return None
        return group.step_device([state], [mask], step_dt, CONFIG["substeps"], plan,
                                 counters=counters, diagnostics=diagnostics,
                                 streams=[stream.cuda_stream])

    # ---- warm-up ----
    for _ in range(args.warmup):
        restore()
        one_step()
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
            one_step()
            e_end[s].record(stream)
            km, nl = C.c_float(), C.c_int()
            lib.fsbm_ctx_last_timing(ctx.handle if group is None else gctx, C.byref(km), C.byref(nl))
            kern_ms.append(km.value)
            launches += nl.value
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        wall = time.perf_counter() - wall0
    step_ms = sum(a.elapsed_time(b) for a, b in zip(e_beg, e_end)) / args.steps
    kernel_ms = sum(kern_ms) / len(kern_ms)
    # diagnostics (the only collective: one NCCL all-reduce of a few scalars); the state
    # keeps this step's output for the parity leg below
    restore()
    if group is None:
        m0 = mass()
        one_step(counters=None)
        m1 = mass()
        diag = shard.reduce_diagnostics(
            shard.StepDiagnostics(cnt.triples // args.steps, cnt.points // args.steps,
                                  cnt.kernel_evals // args.steps, m0.item(), m1.item()), dist, dev)
    else:  # counters and masses already summed over every rank by the library (NCCL)
        gcnt = fsbm.WorkCounters()
        gd = one_step(counters=gcnt, diagnostics=True)
        diag = shard.StepDiagnostics(gcnt.triples, gcnt.points, gcnt.kernel_evals,
                                     float(gd.mass_before.sum()), float(gd.mass_after.sum()))
    tmax = torch.tensor([step_ms, kernel_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)  # device time: max over ranks
    step_ms_max, kernel_ms_max = tmax.tolist()
    points, triples, m0g, m1g = float(diag.points), float(diag.triples), diag.mass_before, diag.mass_after
    value = points / (step_ms_max * 1e-3)

    # ---- roofline (FP64 pipe; algorithmic flops) ----
    peak = fp64_peak(local)
    kname = ctx.fast_kernel() if args.numerics == "fast" else "coal_exact"
    per_rank = world if group is not None else 1  # group counters are summed over ranks
    roof = roofline(nkr, cnt.triples / args.steps / per_rank, cnt.points / args.steps / per_rank,
                    kernel_ms, peak,
                    kname, tag=f"{nkr}-dense" if dense else None)
    roof["kernel_share_of_step"] = kernel_ms / step_ms

    # ---- CPU baseline + parity on a bounded sample (rank 0, N=1 only) ----
    cpu = par = None
    if world == 1 and rank == 0 and not args.no_cpu and not dense:
        try:
            ref = RefCase(nkr)
            cpu, par = sample_parity(fsbm, ctx, grid, ref, (args.ni, args.nk, args.nj), T, P,
                                     pristine, state.bins, args.cpu_seconds, dev)
        except Exception as ex:  # the reference .so may be absent on a stripped tree
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    # ---- EXACT numerics at the same configuration (N=1) ----
    exact = None
    if world == 1 and not args.no_exact and args.numerics == "fast":
        xplan = fsbm.ExecPlan("parallel", 3, 1, "on_demand", "arena", "exact")
        timed_steps(fsbm, lib, ctx, state, mask, xplan, 1, restore, stream, step_dt)
        xs_ms, xk_ms, _, xc = timed_steps(fsbm, lib, ctx, state, mask, xplan, 2, restore, stream,
                                          step_dt)
        exact = {"value": (xc.points / 2) / (xs_ms * 1e-3), "unit": UNIT, "ms_per_step": xs_ms,
                 "steps": 2, "numerics": "exact (bitwise coal_step: reference operation order, "
                                         "no FMA)",
                 "roofline": roofline(nkr, xc.triples / 2, xc.points / 2, xk_ms, peak,
                                      "coal_exact", tag=f"{nkr}-exact"),
                 "bitwise_vs_reference_on_sample": par["exact_bitwise_vs_reference"] if par else None}
        exact["roofline"]["note"] = ("no-FMA reference operation order caps this kernel at half "
                                     "the DFMA roof")

    # ---- e2e through the host C ABI ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, state, pristine, T, P, i0, i1, plan, world, step_dt)

    # ---- the other BASELINE configs (N=1): C3, C4, C5 patch, dense C2 ----
    configs = None
    if world == 1 and not args.no_configs and args.nkr == 33 and not dense:
        del state, pristine, mask
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        configs = {}
        todo = [c for c in args.configs.split(",") if c]
        for lab in todo:
            try:
                if lab == "C3":
                    configs[lab] = run_config(args, "C3", 66, (425, 50, 300), dev, peak)
                elif lab == "C4":
                    configs[lab] = run_config(args, "C4", 132, (425, 50, 300), dev, peak)
                elif lab == "C5":
                    configs[lab] = run_config(args, "C5 per-GPU patch (106 of 850 i-rows)", 264,
                                              (106, 50, 600), dev, peak, steps=2, offset_rows=850)
                elif lab == "C2-cf03":  # SURVEY 8(d)'s imbalance test: scattered cf 0.3 mask
                    configs[lab] = run_config(args, "C2 cloud fraction 0.3", 33, (425, 50, 300), dev,
                                              peak, cf=0.3)
                elif lab == "C2-dense":
                    configs[lab] = run_config(args, "C2 dense input", 33, (425, 50, 300), dev,
                                              peak, dense=True)
                elif lab == "C2-bott":
                    configs[lab] = run_config(args, "C2 Bott", 33, (425, 50, 300), dev, peak,
                                              steps=2, numerics="bott")
            except Exception as ex:
                configs[lab] = {"error": f"{type(ex).__name__}: {ex}"}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (SURVEY 8(d) thunderstorm builder; golovin tables)",
                "config": config_block(args, world),
                "e2e": e2e, "gpu_launches": launches * world,
                "roofline": roof, "cpu_baseline": cpu, "parity": par,
                "clocks": clk.summary(),
                "diagnostics": {"updates_per_step": points, "triples_per_step": triples,
                                "mass_before": m0g, "mass_after": m1g,
                                "mass_rel_drift": abs(m1g - m0g) / m0g, "wall_s_timed": wall},
                "exact": exact, "configs": configs}
        print(json.dumps(line), flush=True)
    if group is not None:
        group.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, ctx, state, pristine, T, P, i0, i1, plan, world, dt=CONFIG["dt"]):
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
    sctx = fsbm.StepContext(ctx, fsbm.CoalConfig(dt, CONFIG["substeps"]), cnt)
    times = []
    for s in range(1 + args.e2e_steps):
        for h, p in zip(host_bins, pristine):  # restore input (not timed)
            h.copy_(p)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        fsbm.fissioned_step(hstate, None, sctx, plan)
        el = time.perf_counter() - t0
        if s > 0:
            times.append(el)
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=state.bins[0].device)
    pts = torch.tensor([float(cnt.points) / (1 + args.e2e_steps)], dtype=torch.float64,
                       device=state.bins[0].device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(pts, op=dist.ReduceOp.SUM)
    h2d = 6 * n * args.nkr * 8 + 2 * n * 8
    d2h = 6 * n * args.nkr * 8
    del host_bins, hT, hP, hstate
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
