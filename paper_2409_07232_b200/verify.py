"""Snapshots and the diffwrf-style comparator: mirror of snapshot.hpp / verify.hpp.

``write_snapshot`` / ``read_snapshot`` keep the reference's CBSNAP01 file format
(snapshot.hpp:8-17) byte for byte; ``compare_states`` runs the digit-agreement
reduction (verify.cpp:12-80) on the GPU (``fsbm_compare_states_device``), uploading
host states first.  Errors follow the reference: ConfigError for bad files,
ShapeError for mismatched states, DomainError for non-finite values.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import ShapeError, fsbm_field_diff, fsbm_ranges
from .coalbench import CATEGORIES, NCAT, GridState, MassGrid, Ranges, _is_cuda, _ptr

__all__ = ["write_snapshot", "read_snapshot", "FieldDiff", "DiffReport", "digit_agreement",
           "compare_states", "format_diff_report"]

FIELDS = ("mass_grid", "temperature", "pressure") + CATEGORIES  # verify.cpp:72-77 order


def _host(a) -> np.ndarray:
    if _is_cuda(a):
        a = a.cpu().numpy()
    return np.ascontiguousarray(a, dtype=np.float64)


def write_snapshot(state: GridState, path: str) -> None:
    """write_snapshot (snapshot.cpp:46-73)."""
    x = _host(state.grid.x)
    T, P = _host(state.temperature), _host(state.pressure)
    bins = [_host(b) for b in state.bins]
    ptrs = (C.c_void_p * NCAT)(*[b.ctypes.data for b in bins])
    _lib.check(_lib.load().fsbm_snapshot_write(str(path).encode(), state.ranges.to_c(), len(x),
                                               float(state.grid.ratio), x.ctypes.data,
                                               T.ctypes.data, P.ctypes.data, ptrs))


def read_snapshot(path: str) -> GridState:
    """read_snapshot (snapshot.cpp:75-135) -> a host GridState."""
    lib = _lib.load()
    r, nkr, ratio = fsbm_ranges(), C.c_int(), C.c_double()
    _lib.check(lib.fsbm_snapshot_read_header(str(path).encode(), C.byref(r), C.byref(nkr),
                                             C.byref(ratio)))
    ranges = Ranges(r.ids, r.ide, r.kds, r.kde, r.jds, r.jde)
    np_ = ranges.npoints()
    x = np.empty(nkr.value)
    T, P = np.empty(np_), np.empty(np_)
    bins = [np.empty(np_ * nkr.value) for _ in range(NCAT)]
    ptrs = (C.c_void_p * NCAT)(*[b.ctypes.data for b in bins])
    _lib.check(lib.fsbm_snapshot_read(str(path).encode(), x.ctypes.data, T.ctypes.data,
                                      P.ctypes.data, ptrs))
    return GridState(ranges, MassGrid(x, ratio.value), T, P, bins)


@dataclass
class FieldDiff:
    """verify.hpp:20-26"""
    field: str
    min_digits: int = 16
    mean_digits: float = 16.0
    count_compared: int = 0
    count_exact: int = 0


@dataclass
class DiffReport:
    """verify.hpp:28-33"""
    fields: list = field(default_factory=list)

    def all_exact(self) -> bool:
        return all(f.count_exact == f.count_compared for f in self.fields)

    def min_digits(self) -> int:
        return min([16] + [f.min_digits for f in self.fields])


def _device_arrays(state: GridState, dev):
    import torch

    def d(a):
        if _is_cuda(a):
            return a.contiguous()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

    return d(state.grid.x), d(state.temperature), d(state.pressure), [d(b) for b in state.bins]


def compare_states(a: GridState, b: GridState, device: int = 0) -> DiffReport:
    """compare_states (verify.cpp:65-80), reduced on the GPU."""
    import torch

    if a.ranges != b.ranges:
        raise ShapeError("compare_states: domain ranges differ")
    if a.nkr() != b.nkr():
        raise ShapeError(f"compare_states: nkr differs ({a.nkr()} vs {b.nkr()})")
    dev = torch.device("cuda", device)
    xa, ta, pa, ba = _device_arrays(a, dev)
    xb, tb, pb, bb = _device_arrays(b, dev)
    out = (fsbm_field_diff * len(FIELDS))()
    stream = torch.cuda.current_stream(dev).cuda_stream
    pa6 = (C.c_void_p * NCAT)(*[t.data_ptr() for t in ba])
    pb6 = (C.c_void_p * NCAT)(*[t.data_ptr() for t in bb])
    _lib.check(_lib.load().fsbm_compare_states_device(
        device, a.ranges.npoints(), a.nkr(), xa.data_ptr(), ta.data_ptr(), pa.data_ptr(), pa6,
        xb.data_ptr(), tb.data_ptr(), pb.data_ptr(), pb6, out, stream))
    return DiffReport([FieldDiff(n, o.min_digits, o.mean_digits, int(o.count_compared),
                                 int(o.count_exact)) for n, o in zip(FIELDS, out)])


def digit_agreement(a: float, b: float, device: int = 0) -> int:
    """digit_agreement (verify.cpp:12-26) of two scalars (a one-value comparator launch)."""
    g = MassGrid(np.array([float(a)]), 2.0)
    h = MassGrid(np.array([float(b)]), 2.0)
    r = Ranges(1, 1, 1, 1, 1, 1)
    z = np.zeros(1)
    sa = GridState(r, g, z, z, [z] * NCAT)
    sb = GridState(r, h, z, z, [z] * NCAT)
    return compare_states(sa, sb, device).fields[0].min_digits


def format_diff_report(report: DiffReport) -> str:
    """format_diff_report (verify.cpp:82-96)."""
    out = "field          min_digits  mean_digits     compared        exact\n"
    for f in report.fields:
        out += f"{f.field:<14} {f.min_digits:10d} {f.mean_digits:12.2f} {f.count_compared:12d} " \
               f"{f.count_exact:12d}\n"
    return out
