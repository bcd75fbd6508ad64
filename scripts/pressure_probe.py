"""coal step time vs the pressure weight (w = 0 / 0.4 / 1 everywhere, and the reference's
900->400 hPa profile) for one grid: how much the per-point K500 + w Kd interpolation costs.
  python scripts/pressure_probe.py <nkr> <ni> <nj> [nk]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_07232_b200 as fsbm  # noqa: E402
from paper_2409_07232_b200 import synth  # noqa: E402

nkr, ni, nj = (int(a) for a in sys.argv[1:4])
nk = int(sys.argv[4]) if len(sys.argv) > 4 else 50
grid = fsbm.make_mass_grid(nkr, 3.35e-14, fsbm.equal_range_ratio(nkr))
tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(), fsbm.KernelParams("golovin", 1.0, 1.5, 0.05))
ctx = fsbm.CoalContext(grid, tabs, 0)
T, P, _ = synth.thermo_host(ni, nk, nj, 1.0, 42, grid)
for label, pv in (("profile", None), ("w=0 (400 hPa)", 400.0), ("w=0.4 (600 hPa)", 600.0), ("w=1 (900 hPa)", 900.0)):
    Pp = P if pv is None else np.full_like(P, pv)
    state, mask = synth.thunderstorm_device(ctx, ni, nk, nj, 1.0, 42, thermo=(T, Pp, None))
    pristine = [b.clone() for b in state.bins]
    s = torch.cuda.current_stream()
    sc = fsbm.StepContext(ctx, stream=s.cuda_stream)
    ms = []
    for it in range(4):
        for b, p0 in zip(state.bins, pristine):
            b.copy_(p0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fsbm.fissioned_step(state, mask, sc, fsbm.ExecPlan())
        e1.record(s)
        torch.cuda.synchronize()
        if it:
            ms.append(e0.elapsed_time(e1))
    npts = ni * nk * nj
    print(f"{nkr} bins {label:>16}: {np.mean(ms):8.2f} ms  {npts / np.mean(ms) / 1e3:8.3f} M upd/s", flush=True)
    del state, mask, pristine
    torch.cuda.empty_cache()
