"""Multi-GPU coalescence step: the C ABI's device groups (include/fsbm_coal.h).

``DeviceGroup`` owns one context per local device; ``step_device`` steps one shard per
device (device-resident state), ``step_host`` splits a host GridState into i-slabs or
WRF-style j-patches (decompose, driver.cpp:187-196) and steps them in place.  Counters,
the first failing point (serial (tile, j, k, i) order) and diagnostics come back reduced
over every shard -- on the host inside a process, by an NCCL all-reduce inside the
library across processes (one group per rank under torchrun; ``nccl_unique_id`` on rank
0, broadcast by the caller).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import fsbm_counters, fsbm_diag, fsbm_error, fsbm_shard, fsbm_tile
from .coalbench import (NCAT, ExecPlan, GridState, KernelTableSet, MassGrid, PatchTilePlan,
                        PredicateMask, Ranges, WorkCounters, _check_buffers, _ptr)
from .shard import decompose_shards

__all__ = ["DeviceGroup", "GroupDiagnostics", "nccl_unique_id", "SPLIT"]

SPLIT = {"i": 0, "j": 1}


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _lib.check(_lib.load().fsbm_nccl_unique_id(buf))
    return bytes(buf.raw)


@dataclass
class GroupDiagnostics:
    number_before: np.ndarray
    number_after: np.ndarray
    mass_before: np.ndarray
    mass_after: np.ndarray
    coal_kernel_ms_max: float


class DeviceGroup:
    """fsbm_group: len(devices) local contexts; this process is `rank` of `nranks`."""

    def __init__(self, grid: MassGrid, tables: KernelTableSet, devices: Sequence[int] = (0,),
                 rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None):
        lib = _lib.load()
        abd = np.array([[p.source_a, p.source_b, p.dest] for p in tables.pairs], np.int32)
        self._keep = [np.ascontiguousarray(grid.x, np.float64), abd.reshape(-1),
                      np.ascontiguousarray(tables.t750, np.float64).reshape(-1),
                      np.ascontiguousarray(tables.t500, np.float64).reshape(-1)]
        devs = (C.c_int * len(devices))(*devices)
        idb = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        h = C.c_void_p()
        _lib.check(lib.fsbm_group_create(len(devices), devs, rank, nranks, idb, grid.nkr(),
                                         self._keep[0].ctypes.data, grid.ratio, len(tables.pairs),
                                         self._keep[1].ctypes.data, self._keep[2].ctypes.data,
                                         self._keep[3].ctypes.data, C.byref(h)))
        self.handle = h
        self.grid = grid
        self.devices = list(devices)
        self.rank, self.nranks = rank, nranks

    def ctx_handle(self, local: int) -> C.c_void_p:
        c = C.c_void_p()
        _lib.check(_lib.load().fsbm_group_ctx(self.handle, local, C.byref(c)))
        return c

    @staticmethod
    def _tiles(tiles: Optional[PatchTilePlan]):
        t = tiles.tiles if tiles is not None else []
        arr = (fsbm_tile * max(1, len(t)))(*[fsbm_tile(*x) for x in t])
        return (arr if t else None), len(t)

    def step_device(self, states: Sequence[GridState], masks: Sequence[Optional[PredicateMask]],
                    dt: float = 1.0, substeps: int = 1, plan: ExecPlan = ExecPlan(),
                    tiles: Optional[PatchTilePlan] = None, counters: Optional[WorkCounters] = None,
                    diagnostics: bool = False, streams: Optional[Sequence[int]] = None):
        """One shard per local device: states[d] holds that shard's device arrays and its
        GLOBAL ranges.  Returns GroupDiagnostics when diagnostics=True."""
        import torch
        if len(states) != len(self.devices):
            raise _lib.ShapeError("step_device: one shard state per local device")
        arr = (fsbm_shard * len(states))()
        for d, st in enumerate(states):
            m = masks[d] if masks else None
            if st.nkr() != self.grid.nkr():
                raise _lib.ShapeError("coal_step: state distribution size does not match nkr")
            if not st.on_device():
                raise _lib.DomainError("step_device: shard state must be device memory")
            _check_buffers(st, m, _Dev(self.devices[d]))
            s = streams[d] if streams else torch.cuda.current_stream(st.bins[0].device).cuda_stream
            arr[d] = fsbm_shard(st.ranges.to_c(), (C.c_void_p * NCAT)(*[_ptr(b) for b in st.bins]),
                                _ptr(st.pressure), _ptr(st.temperature),
                                _ptr(m.call_coal) if m is not None else 0, s)
        tarr, nt = self._tiles(tiles)
        cnt, err, dg = fsbm_counters(), fsbm_error(), fsbm_diag()
        st = _lib.load().fsbm_group_step_device(self.handle, arr, dt, substeps,
                                                C.byref(plan.to_c()), tarr, nt, C.byref(cnt),
                                                C.byref(err), C.byref(dg) if diagnostics else None)
        if counters is not None and st in (0, 4):
            counters.triples += cnt.triples
            counters.points += cnt.points
            counters.kernel_evals += cnt.kernel_evals
        _lib.check(st, err)
        if diagnostics:
            return GroupDiagnostics(np.array(dg.number_before[:]), np.array(dg.number_after[:]),
                                    np.array(dg.mass_before[:]), np.array(dg.mass_after[:]),
                                    float(dg.coal_kernel_ms_max))
        return None

    def step_host(self, state: GridState, mask: Optional[PredicateMask], split: str = "j",
                  dt: float = 1.0, substeps: int = 1, plan: ExecPlan = ExecPlan(),
                  tiles: Optional[PatchTilePlan] = None,
                  counters: Optional[WorkCounters] = None) -> None:
        """fissioned_step on a host GridState: ndev*nranks i-slabs / j-patches, this
        process's shards stepped in place, one host thread per device."""
        if state.on_device():
            raise _lib.DomainError("step_host: state must be host memory")
        if mask is not None and mask.ranges != state.ranges:
            raise _lib.ShapeError("fissioned_step: mask extents do not match the state")
        if state.nkr() != self.grid.nkr():
            raise _lib.ShapeError("coal_step: state distribution size does not match nkr")
        _check_buffers(state, mask, _Dev(self.devices[0]))
        tarr, nt = self._tiles(tiles)
        cnt, err = fsbm_counters(), fsbm_error()
        binsp = (C.c_void_p * NCAT)(*[_ptr(b) for b in state.bins])
        st = _lib.load().fsbm_group_step_host(
            self.handle, state.ranges.to_c(), SPLIT[split], binsp, _ptr(state.pressure),
            _ptr(state.temperature), _ptr(mask.call_coal) if mask is not None else 0, dt,
            substeps, C.byref(plan.to_c()), tarr, nt, C.byref(cnt), C.byref(err))
        if counters is not None and st in (0, 4):
            counters.triples += cnt.triples
            counters.points += cnt.points
            counters.kernel_evals += cnt.kernel_evals
        _lib.check(st, err)

    def last_kernel_ms(self) -> float:
        ms = C.c_float()
        _lib.check(_lib.load().fsbm_group_last_timing(self.handle, C.byref(ms)))
        return ms.value

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().fsbm_group_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Dev:
    """Minimal stand-in for a CoalContext in _check_buffers (only .device is read)."""

    def __init__(self, device: int):
        self.device = device
