"""ctypes binding of the C ABI in include/fsbm_coal.h (libfsbm_coal.so).

There is deliberately no fallback: if the CUDA library is missing or no GPU is
present, every compute entry point raises.  ``load()`` only needs the .so file
(it can be loaded on a CPU-only host to check the exported symbols).
"""
from __future__ import annotations

import ctypes as C
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_PKG, "_lib", "libfsbm_coal.so")
# FSBM_LIB_PATH: load another build of the same C ABI (A/B kernel experiments)
SO_PATH = os.environ.get("FSBM_LIB_PATH", SO_PATH)
HEADER = os.path.join(os.path.dirname(_PKG), "include", "fsbm_coal.h")

NCAT = 6
ABI_VERSION = 2


class fsbm_ranges(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("ids", "ide", "kds", "kde", "jds", "jde")]


class fsbm_plan(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("mode", "collapse", "threads", "kernel_strategy",
                                       "scratch_strategy", "numerics")]


class fsbm_tile(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("its", "ite", "jts", "jte")]


class fsbm_counters(C.Structure):
    _fields_ = [("triples", C.c_uint64), ("points", C.c_uint64), ("kernel_evals", C.c_uint64)]


class fsbm_error(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("category", "bin", "has_point", "i", "k", "j")] + \
        [("value", C.c_double)]


class fsbm_shard(C.Structure):
    _fields_ = [("ranges", fsbm_ranges), ("bins", C.c_void_p * NCAT), ("pressure", C.c_void_p),
                ("temperature", C.c_void_p), ("mask", C.c_void_p), ("stream", C.c_void_p)]


class fsbm_diag(C.Structure):
    _fields_ = [("number_before", C.c_double * NCAT), ("number_after", C.c_double * NCAT),
                ("mass_before", C.c_double * NCAT), ("mass_after", C.c_double * NCAT),
                ("coal_kernel_ms_max", C.c_float)]


class fsbm_field_diff(C.Structure):
    _fields_ = [("min_digits", C.c_int), ("mean_digits", C.c_double),
                ("count_compared", C.c_uint64), ("count_exact", C.c_uint64)]


_vp = C.c_void_p
_SIGS = {
    "fsbm_last_error": ([], C.c_char_p),
    "fsbm_abi_version": ([], C.c_int),
    "fsbm_ctx_create": ([C.c_int, C.c_int, _vp, C.c_double, C.c_int, _vp, _vp, _vp,
                         C.POINTER(_vp)], C.c_int),
    "fsbm_ctx_destroy": ([_vp], C.c_int),
    "fsbm_ctx_gain_table": ([_vp, _vp, _vp, _vp, _vp], C.c_int),
    "fsbm_fission_predicates_device": ([_vp, C.c_size_t, _vp, _vp, C.POINTER(C.c_uint64), _vp],
                                       C.c_int),
    "fsbm_step_grid_device": ([_vp, fsbm_ranges, _vp * NCAT, _vp, _vp, _vp, C.c_double, C.c_int,
                               C.POINTER(fsbm_plan), _vp, C.c_int, _vp,
                               C.POINTER(fsbm_counters), C.POINTER(fsbm_error)], C.c_int),
    "fsbm_step_grid_host": ([_vp, fsbm_ranges, _vp * NCAT, _vp, _vp, _vp, C.c_double, C.c_int,
                             C.POINTER(fsbm_plan), _vp, C.c_int, C.POINTER(fsbm_counters),
                             C.POINTER(fsbm_error)], C.c_int),
    "fsbm_step_patch_host": ([_vp, fsbm_ranges, fsbm_ranges, _vp * NCAT, _vp, _vp, _vp, C.c_double,
                              C.c_int, C.POINTER(fsbm_plan), _vp, C.c_int,
                              C.POINTER(fsbm_counters), C.POINTER(fsbm_error)], C.c_int),
    "fsbm_state_moments_device": ([_vp, C.c_size_t, _vp * NCAT, C.c_double * (2 * NCAT), _vp],
                                  C.c_int),
    "fsbm_decompose": ([fsbm_ranges, C.c_int, C.c_int, C.POINTER(fsbm_ranges)], C.c_int),
    "fsbm_nccl_unique_id": ([C.c_char * 128], C.c_int),
    "fsbm_group_create": ([C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, _vp, C.c_int, _vp,
                           C.c_double, C.c_int, _vp, _vp, _vp, C.POINTER(_vp)], C.c_int),
    "fsbm_group_destroy": ([_vp], C.c_int),
    "fsbm_group_ctx": ([_vp, C.c_int, C.POINTER(_vp)], C.c_int),
    "fsbm_group_step_device": ([_vp, C.POINTER(fsbm_shard), C.c_double, C.c_int,
                                C.POINTER(fsbm_plan), _vp, C.c_int, C.POINTER(fsbm_counters),
                                C.POINTER(fsbm_error), C.POINTER(fsbm_diag)], C.c_int),
    "fsbm_group_step_host": ([_vp, fsbm_ranges, C.c_int, _vp * NCAT, _vp, _vp, _vp, C.c_double,
                              C.c_int, C.POINTER(fsbm_plan), _vp, C.c_int,
                              C.POINTER(fsbm_counters), C.POINTER(fsbm_error)], C.c_int),
    "fsbm_group_last_timing": ([_vp, C.POINTER(C.c_float)], C.c_int),
    "fsbm_coal_step": ([_vp, _vp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                        C.POINTER(fsbm_counters), C.POINTER(fsbm_error)], C.c_int),
    "fsbm_synth_thermo_host": ([C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, _vp,
                                C.c_double, _vp, _vp, _vp], C.c_int),
    "fsbm_synth_thunderstorm_device": ([_vp, C.c_size_t, C.c_uint64, _vp, C.c_uint64,
                                        _vp * NCAT, _vp], C.c_int),
    "fsbm_ctx_last_timing": ([_vp, C.POINTER(C.c_float), C.POINTER(C.c_int)], C.c_int),
    "fsbm_ctx_fast_kernel": ([_vp, C.POINTER(C.c_int)], C.c_int),
    "fsbm_probe_fp64_peak": ([C.c_int, C.POINTER(C.c_double)], C.c_int),
    "fsbm_snapshot_write": ([C.c_char_p, fsbm_ranges, C.c_int, C.c_double, _vp, _vp, _vp,
                             _vp * NCAT], C.c_int),
    "fsbm_snapshot_read_header": ([C.c_char_p, C.POINTER(fsbm_ranges), C.POINTER(C.c_int),
                                   C.POINTER(C.c_double)], C.c_int),
    "fsbm_snapshot_read": ([C.c_char_p, _vp, _vp, _vp, _vp * NCAT], C.c_int),
    "fsbm_compare_states_device": ([C.c_int, C.c_size_t, C.c_int, _vp, _vp, _vp, _vp * NCAT,
                                    _vp, _vp, _vp, _vp * NCAT, C.POINTER(fsbm_field_diff), _vp],
                                   C.c_int),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares (parsed from include/fsbm_coal.h)."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fsbm_[a-z_0-9]+)\s*\(", txt)))


def load(path: str = SO_PATH):
    """Load libfsbm_coal.so (building it first if this tree has nvcc and no .so)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        from . import build as _build
        _build.build()
    lib = C.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.fsbm_abi_version() != ABI_VERSION:
        raise RuntimeError("libfsbm_coal.so ABI version mismatch")
    _lib = lib
    return lib


# ---- error taxonomy (errors.hpp:10-74) ------------------------------------------
class Error(RuntimeError):
    """coalbench::Error"""


class DomainError(Error):
    pass


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class StiffnessError(Error):
    def __init__(self, msg, category=-1, bin=-1, point=None, value=None):
        super().__init__(msg)
        self.category = category
        self.bin = bin
        self.point = point  # (i, k, j) 1-based, or None
        self.value = value  # the negative bin value of the message

    def has_point(self):
        return self.point is not None


class AllocationError(Error):
    pass


class CudaError(Error):
    pass


_STATUS = {1: DomainError, 2: ShapeError, 3: ConfigError, 4: StiffnessError, 5: AllocationError,
           6: CudaError, 7: Error}


def check(status: int, err: fsbm_error | None = None) -> None:
    if status == 0:
        return
    msg = load().fsbm_last_error().decode(errors="replace")
    cls = _STATUS.get(status, Error)
    if cls is StiffnessError:
        point = (err.i, err.k, err.j) if err is not None and err.has_point else None
        raise StiffnessError(msg, err.category if err else -1, err.bin if err else -1, point,
                             err.value if err is not None else None)
    raise cls(msg)
