"""ctypes bindings for the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module.  The product package never does.

Two checkers are exposed:
  * ``Oracle``    -- oracle/_build/liboracle.so, the plain-C restatement
                     (oracle/coal_oracle.c) of the reference hot path.
  * ``Reference`` -- oracle/_ref/libcoalbench_ref.so, the unmodified reference
                     sources compiled with oracle/ref_shim.cpp (oracle/Makefile).
Both use category-major bins arrays: bins[c, point, bin].
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcoalbench_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")

NCAT = 6
CATEGORIES = ("liquid", "ice1", "ice2", "ice3", "snow", "graupel")


def build(ref: bool = True) -> None:
    """make -C oracle (the restatement always; the reference when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def equal_range_ratio(nkr: int) -> float:
    """ratio = 2^(32/(nkr-1)); exactly 2.0 at 33 bins."""
    return float(2.0 ** (32.0 / (nkr - 1)))


class Oracle:
    """The C restatement (oracle/coal_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.orc_mass_grid.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.orc_exponential_init.argtypes = [C.c_int, _dp, C.c_double, C.c_double, _dp]
        L.orc_gain_table.argtypes = [C.c_int, _dp, C.c_double, _ip, _dp, _dp, _dp]
        L.orc_default_registry.argtypes = [_ip]
        L.orc_build_tables.argtypes = [C.c_int, _dp, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_double, _dp, _dp]
        L.orc_pressure_weight.argtypes = [C.c_double]
        L.orc_pressure_weight.restype = C.c_double
        L.orc_interpolate.argtypes = [C.c_double, C.c_double, C.c_double]
        L.orc_interpolate.restype = C.c_double
        L.orc_coal_step.argtypes = [C.c_int, _dp, C.c_int, _ip, _dp, _dp, _ip, _dp, _dp, _dp,
                                    C.POINTER(C.c_void_p), C.c_double, C.c_double, C.c_int,
                                    C.c_int, _u64p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_splitmix_next.restype = C.c_uint64
        L.orc_uniform01.argtypes = [C.POINTER(C.c_uint64)]
        L.orc_uniform01.restype = C.c_double
        L.orc_synthetic_case.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                         C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp,
                                         C.c_void_p]
        L.orc_thunderstorm_point.argtypes = [C.c_int, _dp, C.c_uint64, C.c_uint64, _dp]
        L.orc_thunderstorm_block.argtypes = [C.c_int, _dp, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_void_p, _dp]
        L.orc_fission_predicates.argtypes = [C.c_uint64, _dp, _u8p]
        L.orc_fission_predicates.restype = C.c_uint64
        L.orc_bott_courant.argtypes = [C.c_int, _dp, _ip, _dp]
        L.orc_bott_flux.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double]
        L.orc_bott_flux.restype = C.c_double
        L.orc_bott_step.argtypes = [C.c_int, _dp, C.c_int, _ip, _dp, _dp, _ip, _dp,
                                    C.POINTER(C.c_void_p), C.c_double, C.c_double, C.c_int,
                                    C.c_int, _u64p]
        L.orc_bott_step_grid.argtypes = [C.c_size_t, C.c_int, _dp, C.c_int, _ip, _dp, _dp, _ip,
                                         _dp, C.c_void_p, _dp, _dp, C.c_double, C.c_int, C.c_int,
                                         C.c_int, _u64p]
        L.orc_step_grid.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_int, _ip, _dp,
                                    _dp, _ip, _dp, _dp, _dp, _u8p, _dp, _dp, C.c_double, C.c_int,
                                    C.c_int, C.c_int, _u64p, _ip]

    def mass_grid(self, nkr, x1=3.35e-14, ratio=2.0):
        x = np.zeros(nkr)
        st = self.lib.orc_mass_grid(nkr, x1, ratio, x)
        if st:
            raise ValueError(f"mass_grid status {st}")
        return x

    def exponential_init(self, x, n_total, xbar):
        out = np.zeros(len(x))
        st = self.lib.orc_exponential_init(len(x), x, n_total, xbar, out)
        if st:
            raise ValueError(f"exponential_init status {st}")
        return out

    def gain_table(self, x, ratio):
        n = len(x)
        lo = np.zeros(n * n, np.int32)
        wlo, whi, top = np.zeros(n * n), np.zeros(n * n), np.zeros(n * n)
        st = self.lib.orc_gain_table(n, x, ratio, lo, wlo, whi, top)
        if st:
            raise ValueError(f"gain_table status {st}")
        return lo, wlo, whi, top

    def default_registry(self):
        abd = np.zeros(60, np.int32)
        self.lib.orc_default_registry(abd)
        return abd

    def build_tables(self, x, npairs=20, family=1, coeff=1.0, level_scale=1.5,
                     pair_scale_step=0.0):
        n = len(x)
        t750 = np.zeros(npairs * n * n)
        t500 = np.zeros(npairs * n * n)
        st = self.lib.orc_build_tables(n, x, npairs, family, coeff, level_scale,
                                       pair_scale_step, t750, t500)
        if st:
            raise ValueError(f"build_tables status {st}")
        return t750, t500

    def pressure_weight(self, p):
        return self.lib.orc_pressure_weight(p)

    def interpolate(self, k750, k500, w):
        return self.lib.orc_interpolate(k750, k500, w)

    def coal_step(self, x, abd, t750, t500, gains, bins6, pressure, dt=1.0, substeps=1,
                  kernel_strategy=1):
        """bins6: (6, nkr) float64 array, updated in place. Returns (status, counters, err)."""
        nkr = len(x)
        assert bins6.shape == (NCAT, nkr) and bins6.flags.c_contiguous
        ptrs = (C.c_void_p * NCAT)(*[bins6[c].ctypes.data for c in range(NCAT)])
        cnt = np.zeros(3, np.uint64)
        ec, eb = C.c_int(-1), C.c_int(-1)
        lo, wlo, whi, top = gains
        st = self.lib.orc_coal_step(nkr, x, len(abd) // 3, abd, t750, t500, lo, wlo, whi, top,
                                    ptrs, pressure, dt, substeps, kernel_strategy, cnt,
                                    C.byref(ec), C.byref(eb))
        return st, cnt, (ec.value, eb.value)

    # ---- Bott (1998) flux method (oracle/bott_oracle.c; parity unpinned: KAT-pinned) ----
    def bott_courant(self, x, lo):
        nkr = len(x)
        cour = np.zeros(nkr * nkr)
        assert self.lib.orc_bott_courant(nkr, x, np.ascontiguousarray(lo, np.int32), cour) == 0
        return cour

    def bott_flux(self, gsk, gk, gkp, c):
        return self.lib.orc_bott_flux(gsk, gk, gkp, c)

    def bott_step(self, x, abd, t750, t500, lo, cour, bins6, pressure, dt=1.0, substeps=1,
                  kernel_strategy=1):
        """bins6: (6, nkr) float64, updated in place.  Returns (status, counters)."""
        nkr = len(x)
        assert bins6.shape == (NCAT, nkr) and bins6.flags.c_contiguous
        ptrs = (C.c_void_p * NCAT)(*[bins6[c].ctypes.data for c in range(NCAT)])
        cnt = np.zeros(3, np.uint64)
        st = self.lib.orc_bott_step(nkr, x, len(abd) // 3, abd, t750, t500,
                                    np.ascontiguousarray(lo, np.int32), cour, ptrs, pressure, dt,
                                    substeps, kernel_strategy, cnt)
        return st, cnt

    def bott_step_grid(self, x, abd, t750, t500, lo, cour, mask, P, bins, dt=1.0, substeps=1,
                       kernel_strategy=1, threads=None):
        """bins: category-major (6, np, nkr) float64, updated in place.  Returns (st, counters)."""
        nkr = len(x)
        npt = bins.shape[1]
        assert bins.shape == (NCAT, npt, nkr) and bins.flags.c_contiguous
        cnt = np.zeros(3, np.uint64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        st = self.lib.orc_bott_step_grid(npt, nkr, x, len(abd) // 3, abd, t750, t500,
                                         np.ascontiguousarray(lo, np.int32), cour,
                                         None if m is None else m.ctypes.data,
                                         np.ascontiguousarray(P, np.float64), bins, dt, substeps,
                                         kernel_strategy, threads or os.cpu_count() or 1, cnt)
        return st, cnt

    def synthetic_case(self, ni, nk, nj, cloud_fraction, seed, nkr=33, x1=3.35e-14, ratio=2.0,
                       number_density=1e6, spectra=True):
        """make_synthetic_case restated; spectra=False returns (T, P, None) without
        allocating the 6 x npoints x nkr liquid-only spectra (same T/P bytes)."""
        np_ = ni * nk * nj
        T, P = np.zeros(np_), np.zeros(np_)
        bins = np.zeros(NCAT * np_ * nkr) if spectra else None
        st = self.lib.orc_synthetic_case(ni, nk, nj, cloud_fraction, seed, nkr, x1, ratio,
                                         number_density, T, P,
                                         bins.ctypes.data if spectra else None)
        if st:
            raise ValueError(f"synthetic_case status {st}")
        return T, P, (bins.reshape(NCAT, np_, nkr) if spectra else None)

    def thunderstorm_point(self, x, seed, p):
        out = np.zeros(NCAT * len(x))
        st = self.lib.orc_thunderstorm_point(len(x), x, seed, p, out)
        if st:
            raise ValueError(f"thunderstorm_point status {st}")
        return out.reshape(NCAT, len(x))

    def thunderstorm_block(self, x, seed, p0, n, mask=None):
        out = np.zeros(NCAT * n * len(x))
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        st = self.lib.orc_thunderstorm_block(len(x), x, seed, p0, n,
                                             None if m is None else m.ctypes.data, out)
        if st:
            raise ValueError(f"thunderstorm_block status {st}")
        return out.reshape(NCAT, n, len(x))

    def fission_predicates(self, T):
        mask = np.zeros(len(T), np.uint8)
        n = self.lib.orc_fission_predicates(len(T), np.ascontiguousarray(T), mask)
        return mask, int(n)

    def step_grid(self, ni, nk, nj, x, abd, t750, t500, gains, mask, P, bins, dt=1.0,
                  substeps=1, kernel_strategy=1, nthreads=1):
        """bins: (6, npoints, nkr) float64, updated in place."""
        nkr = len(x)
        cnt = np.zeros(3, np.uint64)
        err = np.full(5, -1, np.int32)
        lo, wlo, whi, top = gains
        st = self.lib.orc_step_grid(ni, nk, nj, nkr, x, len(abd) // 3, abd, t750, t500, lo, wlo,
                                    whi, top, mask, P, bins.reshape(-1), dt, substeps,
                                    kernel_strategy, nthreads, cnt, err)
        return st, cnt, err


class Reference:
    """The unmodified reference library (oracle/_ref/libcoalbench_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.cbref_last_error.restype = C.c_char_p
        L.cbref_default_registry.argtypes = [_ip]
        L.cbref_mass_grid.argtypes = [C.c_int, C.c_double, C.c_double, _dp]
        L.cbref_gain_table.argtypes = [C.c_int, C.c_double, C.c_double, _ip, _dp, _dp, _dp]
        L.cbref_build_tables.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_void_p,
                                         C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.cbref_exponential_init.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                             C.c_double, _dp]
        L.cbref_pressure_weight.argtypes = [C.c_double]
        L.cbref_pressure_weight.restype = C.c_double
        L.cbref_kernel_at.argtypes = [C.c_int, C.c_int, C.c_void_p, _dp, _dp, C.c_int, C.c_int,
                                      C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.cbref_coal_step.argtypes = [C.c_int, C.c_double, C.c_double, C.c_int, C.c_void_p, _dp,
                                      _dp, _dp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                      _u64p, _ip]
        L.cbref_synthetic_case.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                           C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp,
                                           _dp]
        L.cbref_fission_predicates.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _u8p, _u64p]
        for name in ("cbref_write_snapshot", "cbref_read_snapshot", "cbref_compare_states"):
            getattr(L, name).restype = C.c_int
        L.cbref_write_snapshot.argtypes = [C.c_char_p, C.c_void_p, C.c_int, C.c_double,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.cbref_read_snapshot.argtypes = [C.c_char_p] + [C.c_void_p] * 7
        L.cbref_compare_states.argtypes = [C.c_void_p] + [C.c_int] + [C.c_void_p] * 12
        L.cbref_digit_agreement.argtypes = [C.c_double, C.c_double, C.c_void_p]
        L.cbref_fissioned_step.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                           C.c_double, C.c_int, C.c_void_p, _dp, _dp, _dp, _dp,
                                           _dp, C.c_double, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, C.c_int, _u64p, _dp, _ip]

    def last_error(self) -> str:
        return self.lib.cbref_last_error().decode()

    @staticmethod
    def _abd(abd):
        if abd is None:
            return 20, None
        abd = np.ascontiguousarray(abd, np.int32)
        return len(abd) // 3, abd.ctypes.data

    def default_registry(self):
        abd = np.zeros(60, np.int32)
        self.lib.cbref_default_registry(abd)
        return abd

    def mass_grid(self, nkr, x1=3.35e-14, ratio=2.0):
        x = np.zeros(nkr)
        st = self.lib.cbref_mass_grid(nkr, x1, ratio, x)
        if st:
            raise ValueError(self.last_error())
        return x

    def gain_table(self, nkr, x1=3.35e-14, ratio=2.0):
        lo = np.zeros(nkr * nkr, np.int32)
        wlo, whi, top = np.zeros(nkr * nkr), np.zeros(nkr * nkr), np.zeros(nkr * nkr)
        st = self.lib.cbref_gain_table(nkr, x1, ratio, lo, wlo, whi, top)
        if st:
            raise ValueError(self.last_error())
        return lo, wlo, whi, top

    def build_tables(self, nkr, x1=3.35e-14, ratio=2.0, abd=None, family=1, coeff=1.0,
                     level_scale=1.5, pair_scale_step=0.0):
        npairs, ptr = self._abd(abd)
        t750 = np.zeros(npairs * nkr * nkr)
        t500 = np.zeros(npairs * nkr * nkr)
        st = self.lib.cbref_build_tables(nkr, x1, ratio, npairs, ptr, family, coeff, level_scale,
                                         pair_scale_step, t750, t500)
        if st:
            raise ValueError(self.last_error())
        return t750, t500

    def exponential_init(self, nkr, n_total, xbar, x1=3.35e-14, ratio=2.0):
        out = np.zeros(nkr)
        st = self.lib.cbref_exponential_init(nkr, x1, ratio, n_total, xbar, out)
        if st:
            raise ValueError(self.last_error())
        return out

    def pressure_weight(self, p):
        return self.lib.cbref_pressure_weight(p)

    def kernel_at(self, nkr, t750, t500, pair, i, j, pressure, abd=None):
        npairs, ptr = self._abd(abd)
        out = C.c_double()
        st = self.lib.cbref_kernel_at(nkr, npairs, ptr, t750, t500, pair, i, j, pressure,
                                      C.byref(out))
        if st:
            raise ValueError(self.last_error())
        return out.value

    def coal_step(self, nkr, t750, t500, bins6, pressure, dt=1.0, substeps=1, kernel_strategy=1,
                  scratch_strategy=0, x1=3.35e-14, ratio=2.0, abd=None):
        """bins6: (6, nkr) updated in place. Returns (status, counters, (cat, bin))."""
        npairs, ptr = self._abd(abd)
        cnt = np.zeros(3, np.uint64)
        err = np.full(2, -1, np.int32)
        st = self.lib.cbref_coal_step(nkr, x1, ratio, npairs, ptr, t750, t500,
                                      bins6.reshape(-1), pressure, dt, substeps, kernel_strategy,
                                      scratch_strategy, cnt, err)
        return st, cnt, (int(err[0]), int(err[1]))

    # ---- Bott (1998) flux method (oracle/bott_oracle.c; parity unpinned: KAT-pinned) ----
    def bott_courant(self, x, lo):
        nkr = len(x)
        cour = np.zeros(nkr * nkr)
        assert self.lib.orc_bott_courant(nkr, x, np.ascontiguousarray(lo, np.int32), cour) == 0
        return cour

    def bott_flux(self, gsk, gk, gkp, c):
        return self.lib.orc_bott_flux(gsk, gk, gkp, c)

    def bott_step(self, x, abd, t750, t500, lo, cour, bins6, pressure, dt=1.0, substeps=1,
                  kernel_strategy=1):
        """bins6: (6, nkr) float64, updated in place.  Returns (status, counters)."""
        nkr = len(x)
        assert bins6.shape == (NCAT, nkr) and bins6.flags.c_contiguous
        ptrs = (C.c_void_p * NCAT)(*[bins6[c].ctypes.data for c in range(NCAT)])
        cnt = np.zeros(3, np.uint64)
        st = self.lib.orc_bott_step(nkr, x, len(abd) // 3, abd, t750, t500,
                                    np.ascontiguousarray(lo, np.int32), cour, ptrs, pressure, dt,
                                    substeps, kernel_strategy, cnt)
        return st, cnt

    def bott_step_grid(self, x, abd, t750, t500, lo, cour, mask, P, bins, dt=1.0, substeps=1,
                       kernel_strategy=1, threads=None):
        """bins: category-major (6, np, nkr) float64, updated in place.  Returns (st, counters)."""
        nkr = len(x)
        npt = bins.shape[1]
        assert bins.shape == (NCAT, npt, nkr) and bins.flags.c_contiguous
        cnt = np.zeros(3, np.uint64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        st = self.lib.orc_bott_step_grid(npt, nkr, x, len(abd) // 3, abd, t750, t500,
                                         np.ascontiguousarray(lo, np.int32), cour,
                                         None if m is None else m.ctypes.data,
                                         np.ascontiguousarray(P, np.float64), bins, dt, substeps,
                                         kernel_strategy, threads or os.cpu_count() or 1, cnt)
        return st, cnt

    def synthetic_case(self, ni, nk, nj, cloud_fraction, seed, nkr=33, x1=3.35e-14, ratio=2.0,
                       number_density=1e6):
        np_ = ni * nk * nj
        T, P = np.zeros(np_), np.zeros(np_)
        bins = np.zeros(NCAT * np_ * nkr)
        st = self.lib.cbref_synthetic_case(ni, nk, nj, cloud_fraction, seed, nkr, x1, ratio,
                                           number_density, T, P, bins)
        if st:
            raise ValueError(self.last_error())
        return T, P, bins.reshape(NCAT, np_, nkr)

    def fission_predicates(self, ni, nk, nj, T):
        mask = np.zeros(ni * nk * nj, np.uint8)
        cnt = np.zeros(1, np.uint64)
        st = self.lib.cbref_fission_predicates(ni, nk, nj, np.ascontiguousarray(T), mask, cnt)
        if st:
            raise ValueError(self.last_error())
        return mask, int(cnt[0])

    def fissioned_step(self, ni, nk, nj, nkr, t750, t500, T, P, bins, dt=1.0, substeps=1,
                       mode=1, collapse=3, threads=1, kernel_strategy=1, scratch_strategy=1,
                       n_patches=1, n_tiles=1, x1=3.35e-14, ratio=2.0, abd=None):
        """bins: (6, npoints, nkr), updated in place. Returns (status, counters, timings, err5)."""
        npairs, ptr = self._abd(abd)
        cnt = np.zeros(3, np.uint64)
        tim = np.zeros(2)
        err = np.full(5, -1, np.int32)
        st = self.lib.cbref_fissioned_step(ni, nk, nj, nkr, x1, ratio, npairs, ptr, t750, t500,
                                           np.ascontiguousarray(T), np.ascontiguousarray(P),
                                           bins.reshape(-1), dt, substeps, mode, collapse,
                                           threads, kernel_strategy, scratch_strategy, n_patches,
                                           n_tiles, cnt, tim, err)
        return st, cnt, tim, err

    # ---- snapshot.cpp / verify.cpp (reference state I/O and comparator) ----
    def write_snapshot(self, path, ranges, x, ratio, T, P, bins):
        """bins: (6, npoints*nkr) or (6, npoints, nkr)."""
        L = self.lib
        rg = np.ascontiguousarray(ranges, np.int32)
        x = np.ascontiguousarray(x, np.float64)
        st = L.cbref_write_snapshot(str(path).encode(), rg.ctypes.data, len(x), C.c_double(ratio),
                                    x.ctypes.data, np.ascontiguousarray(T).ctypes.data,
                                    np.ascontiguousarray(P).ctypes.data,
                                    np.ascontiguousarray(bins, np.float64).ctypes.data)
        return st

    def read_snapshot(self, path):
        """Returns (status, ranges[6], x, ratio, T, P, bins (6, np*nkr))."""
        L = self.lib
        rg = np.zeros(6, np.int32)
        nkr, ratio = C.c_int(), C.c_double()
        st = L.cbref_read_snapshot(str(path).encode(), rg.ctypes.data, C.byref(nkr), C.byref(ratio),
                                   None, None, None, None)
        if st:
            return st, None, None, None, None, None, None
        np_ = int((rg[1] - rg[0] + 1) * (rg[3] - rg[2] + 1) * (rg[5] - rg[4] + 1))
        x, T, P = np.zeros(nkr.value), np.zeros(np_), np.zeros(np_)
        bins = np.zeros((NCAT, np_ * nkr.value))
        st = L.cbref_read_snapshot(str(path).encode(), rg.ctypes.data, C.byref(nkr), C.byref(ratio),
                                   x.ctypes.data, T.ctypes.data, P.ctypes.data, bins.ctypes.data)
        return st, rg, x, ratio.value, T, P, bins

    def digit_agreement(self, a, b):
        d = C.c_int()
        st = self.lib.cbref_digit_agreement(C.c_double(a), C.c_double(b), C.byref(d))
        return st, d.value

    def compare_states(self, ranges, xa, Ta, Pa, binsa, xb, Tb, Pb, binsb):
        """Per field (9): (min_digits, mean_digits, count_compared, count_exact)."""
        rg = np.ascontiguousarray(ranges, np.int32)
        mn, mean = np.zeros(9, np.int32), np.zeros(9)
        cmp_, ex = np.zeros(9, np.uint64), np.zeros(9, np.uint64)
        c = lambda a: np.ascontiguousarray(a, np.float64).ctypes.data
        st = self.lib.cbref_compare_states(rg.ctypes.data, len(xa), c(xa), c(Ta), c(Pa), c(binsa),
                                           c(xb), c(Tb), c(Pb), c(binsb), mn.ctypes.data,
                                           mean.ctypes.data, cmp_.ctypes.data, ex.ctypes.data)
        return st, [(int(mn[f]), float(mean[f]), int(cmp_[f]), int(ex[f])) for f in range(9)]
