"""Synthetic atmospheric columns for benches and parity fixtures (not part of the step).

* ``thermo_host`` -- make_synthetic_case's temperature / pressure / cloud mask recipe
  (proj/src/driver.cpp:223-285, SplitMix64 Fisher-Yates) and, optionally, its
  liquid-only spectra, computed by the C++ host library.
* ``thunderstorm_device`` -- SURVEY 8(d) headline input: the same T/P/mask plus all
  six categories populated at every mask-true point, generated on the GPU from a
  counter-based SplitMix64(seed ^ point) so any shard is generated independently.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .coalbench import (CoalContext, GridState, MassGrid, NCAT, PredicateMask, Ranges,
                        fission_predicates)


def thermo_host(ni, nk, nj, cloud_fraction, seed, grid: MassGrid | None = None,
                number_density=1e6, liquid=False):
    np_ = ni * nk * nj
    T = np.zeros(np_)
    P = np.zeros(np_)
    liq = np.zeros(np_ * grid.nkr()) if (liquid and grid is not None) else None
    x = np.ascontiguousarray(grid.x) if grid is not None else None
    st = _lib.load().fsbm_synth_thermo_host(
        ni, nk, nj, cloud_fraction, seed, grid.nkr() if grid is not None else 2,
        x.ctypes.data if x is not None else None, number_density, T.ctypes.data, P.ctypes.data,
        liq.ctypes.data if liq is not None else None)
    _lib.check(st)
    return T, P, liq


def liquid_case_host(ni, nk, nj, cloud_fraction, seed, grid: MassGrid) -> GridState:
    """make_synthetic_case (driver.cpp:223-285) as host numpy arrays."""
    T, P, liq = thermo_host(ni, nk, nj, cloud_fraction, seed, grid, liquid=True)
    bins = [liq] + [np.zeros_like(liq) for _ in range(NCAT - 1)]
    return GridState(Ranges(1, ni, 1, nk, 1, nj), grid, T, P, bins)


def thunderstorm_device(ctx: CoalContext, ni, nk, nj, cloud_fraction=1.0, seed=42,
                        device="cuda:0", i_slab=None, thermo=None):
    """Headline input on device: returns (GridState of CUDA tensors, PredicateMask).

    i_slab=(i0, i1) (0-based, half-open) keeps only that slab of the (ni, nk, nj)
    domain -- one rank's shard; the bytes equal the same slice of the full domain."""
    import torch

    T, P, _ = thermo if thermo is not None else thermo_host(ni, nk, nj, cloud_fraction, seed,
                                                             ctx.grid)
    i0, i1 = i_slab if i_slab is not None else (0, ni)
    per_i = nk * nj
    T = np.ascontiguousarray(T[i0 * per_i:i1 * per_i])
    P = np.ascontiguousarray(P[i0 * per_i:i1 * per_i])
    offset = i0 * per_i
    ni = i1 - i0
    np_ = ni * nk * nj
    dev = torch.device(device)
    Td = torch.from_numpy(T).to(dev)
    Pd = torch.from_numpy(P).to(dev)
    bins = [torch.empty(np_ * ctx.nkr, dtype=torch.float64, device=dev) for _ in range(NCAT)]
    state = GridState(Ranges(1 + i0, i1, 1, nk, 1, nj), ctx.grid, Td, Pd, bins)
    mask = fission_predicates(state, ctx)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ptrs = (C.c_void_p * NCAT)(*[b.data_ptr() for b in bins])
    _lib.check(_lib.load().fsbm_synth_thunderstorm_device(ctx.handle, np_, offset,
                                                          mask.call_coal.data_ptr(), seed, ptrs,
                                                          stream))
    return state, mask
