"""Host-side mirror of the reference's coalbench interface for the hot path.

Names, argument meaning and error behaviour follow /root/reference/proj/include/
coalbench/{mass_grid,kernels,coalescence,driver,errors}.hpp so that code (and
tests) written against the reference read the same; the arithmetic runs in the
sm_100a kernels behind the C ABI (include/fsbm_coal.h).  State may be host
numpy arrays (``fissioned_step`` then goes through ``fsbm_step_grid_host``) or
CUDA torch tensors (``fsbm_step_grid_device``; torch is only used as the
device-memory container).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (AllocationError, ConfigError, CudaError, DomainError, Error, ShapeError,
                   StiffnessError, fsbm_counters, fsbm_error, fsbm_plan, fsbm_ranges, fsbm_tile)

__all__ = [
    "CATEGORIES", "NCAT", "MassGrid", "make_mass_grid", "exponential_init", "total_mass",
    "total_number", "InteractionPair", "default_pair_registry", "KernelParams",
    "KernelTableSet", "build_tables", "validate_registry", "pressure_weight", "interpolate_kernel", "CoalConfig",
    "ExecPlan", "Ranges", "GridState", "PredicateMask", "PatchTilePlan", "decompose",
    "WorkCounters", "PhaseTimings", "StepContext", "CoalContext", "fission_predicates",
    "fissioned_step", "coal_step", "Error", "DomainError", "ShapeError", "ConfigError",
    "StiffnessError", "AllocationError", "CudaError", "equal_range_ratio",
]

CATEGORIES = ("liquid", "ice1", "ice2", "ice3", "snow", "graupel")  # kernels.hpp:17-26
NCAT = 6
OUTER_GATE_K = 193.15  # driver.hpp:17-20
COAL_GATE_K = 223.15


# ---- L0: mass grid (mass_grid.hpp/.cpp) ------------------------------------------
@dataclass
class MassGrid:
    x: np.ndarray
    ratio: float = 2.0

    def nkr(self) -> int:
        return len(self.x)


def make_mass_grid(nkr: int, x1: float = 3.35e-14, ratio: float = 2.0) -> MassGrid:
    """x[k] = x1 * ratio^k by repeated multiplication (mass_grid.cpp:10-25)."""
    if nkr < 2:
        raise DomainError(f"make_mass_grid: nkr must be >= 2, got {nkr}")
    if not (x1 > 0.0) or not math.isfinite(x1):
        raise DomainError("make_mass_grid: x1 must be positive and finite")
    if not (ratio > 1.0) or not math.isfinite(ratio):
        raise DomainError("make_mass_grid: ratio must be > 1")
    x = [float(x1)]
    for _ in range(1, nkr):
        x.append(x[-1] * ratio)
    return MassGrid(np.array(x, dtype=np.float64), float(ratio))


def equal_range_ratio(nkr: int) -> float:
    """2^(32/(nkr-1)) keeps the 33-bin mass range at any nkr (2.0 at 33)."""
    return float(2.0 ** (32.0 / (nkr - 1)))


def exponential_init(grid: MassGrid, n_total: float, xbar: float) -> np.ndarray:
    """mass_grid.cpp:27-48 (host setup helper)."""
    if not (n_total >= 0.0) or not math.isfinite(n_total):
        raise DomainError("exponential_init: n_total must be >= 0")
    if not (xbar > 0.0) or not math.isfinite(xbar):
        raise DomainError("exponential_init: xbar must be > 0")
    n = np.zeros(grid.nkr())
    if n_total == 0.0:
        return n
    wsum = 0.0
    for k, xk in enumerate(grid.x):
        n[k] = xk * math.exp(-xk / xbar)
        wsum += n[k]
    if wsum == 0.0:
        raise DomainError("exponential_init: all weights underflowed to zero")
    return n_total * (n / wsum)


def total_mass(n: np.ndarray, grid: MassGrid) -> float:
    if len(n) != grid.nkr():
        raise ShapeError("total_mass: distribution/grid bin mismatch")
    return float(math.fsum(np.asarray(n) * grid.x))


def total_number(n: np.ndarray) -> float:
    return float(math.fsum(np.asarray(n)))


# ---- L1: registry + tables (kernels.hpp/.cpp) --------------------------------------
@dataclass(frozen=True)
class InteractionPair:
    id: str
    source_a: int
    source_b: int
    dest: int

    def is_self(self) -> bool:
        return self.source_a == self.source_b


def default_pair_registry() -> list[InteractionPair]:
    """The canonical 20 pairs in normative order (kernels.cpp:65-93)."""
    L, I1, I2, I3, S, G = range(6)
    spec = [("cwll", L, L, L), ("cwi1i1", I1, I1, I1), ("cwi2i2", I2, I2, I2),
            ("cwi3i3", I3, I3, I3), ("cwss", S, S, S), ("cwgg", G, G, G),
            ("cwli1", L, I1, I1), ("cwli2", L, I2, I2), ("cwli3", L, I3, I3),
            ("cwls", L, S, S), ("cwlg", L, G, G), ("cwi1s", I1, S, S), ("cwi2s", I2, S, S),
            ("cwi3s", I3, S, S), ("cwi1g", I1, G, G), ("cwi2g", I2, G, G),
            ("cwi3g", I3, G, G), ("cwsg", S, G, G), ("cwsl", S, L, G), ("cwgl", G, L, G)]
    return [InteractionPair(*t) for t in spec]


def validate_registry(pairs: Sequence[InteractionPair], allow_nonstandard_count=False) -> None:
    """kernels.cpp:95-109"""
    if not pairs:
        raise ConfigError("pair registry is empty")
    ids = set()
    for p in pairs:
        if not p.id:
            raise ConfigError("pair registry entry has an empty id")
        if p.id in ids:
            raise ConfigError(f"duplicate pair id '{p.id}' in registry")
        ids.add(p.id)
    if not allow_nonstandard_count and len(pairs) != 20:
        raise ConfigError(f"pair registry has {len(pairs)} entries; 20 required unless "
                          "explicitly overridden")


FAMILIES = {"constant": 0, "golovin": 1, "product": 2, "hydrodynamic": 3}


@dataclass
class KernelParams:
    family: str = "golovin"
    coeff: float = 1.0
    level_scale: float = 1.5
    pair_scale_step: float = 0.0


@dataclass
class KernelTableSet:
    """Per-pair nkr x nkr tables at 750/500 hPa, [pair][i][j] (kernels.hpp:81-114)."""
    pairs: list
    t750: np.ndarray
    t500: np.ndarray

    def nkr(self) -> int:
        return self.t750.shape[-1]

    def num_pairs(self) -> int:
        return len(self.pairs)


def _family_value(fam: int, coeff: float, xi: float, xj: float) -> float:
    if fam == 0:
        return coeff
    if fam == 1:
        return coeff * (xi + xj)
    if fam == 2:
        return coeff * xi * xj
    ri, rj = np.cbrt(xi), np.cbrt(xj)
    sigma = (ri + rj) * (ri + rj)
    return coeff * sigma * math.sqrt(ri * ri + rj * rj)


def build_tables(grid: MassGrid, pairs: Sequence[InteractionPair],
                 params: KernelParams = KernelParams()) -> KernelTableSet:
    """kernels.cpp:117-140 (host-side setup; uploaded once by CoalContext)."""
    for name, v in (("coeff", params.coeff), ("level_scale", params.level_scale),
                    ("pair_scale_step", params.pair_scale_step)):
        if not (v >= 0.0) or not math.isfinite(v):
            raise DomainError(f"build_tables: {name} must be finite and >= 0")
    if params.family not in FAMILIES:
        raise DomainError("build_tables: unknown kernel family")
    validate_registry(pairs, allow_nonstandard_count=True)
    fam = FAMILIES[params.family]
    n = grid.nkr()
    t750 = np.zeros((len(pairs), n, n))
    t500 = np.zeros((len(pairs), n, n))
    base = np.array([[_family_value(fam, params.coeff, float(xi), float(xj)) for xj in grid.x]
                     for xi in grid.x])
    for p in range(len(pairs)):
        v = base * (1.0 + params.pair_scale_step * p)
        t750[p] = v
        t500[p] = v * params.level_scale
    return KernelTableSet(list(pairs), t750, t500)


def pressure_weight(p: float) -> float:
    """kernels.hpp:123-129"""
    w = (p - 500.0) / (750.0 - 500.0)
    return min(max(w, 0.0), 1.0)


def interpolate_kernel(k750: float, k500: float, w: float) -> float:
    """kernels.hpp:133-135 (normative order)."""
    return k500 + (k750 - k500) * w


# ---- L2/L3 configuration types ----------------------------------------------------
PRECOMPUTED, ON_DEMAND = 0, 1
AUTOMATIC, ARENA = 0, 1
FAST, EXACT = 0, 1
_KSTRAT = {"precomputed": 0, "on_demand": 1}
_SSTRAT = {"automatic": 0, "arena": 1}
_NUM = {"fast": 0, "exact": 1, "bott": 2}


@dataclass
class CoalConfig:
    """coalescence.hpp:32-37"""
    dt: float = 1.0
    substeps: int = 1
    kernel_strategy: str = "on_demand"
    scratch_strategy: str = "automatic"


@dataclass
class ExecPlan:
    """driver.hpp:103-109 plus the numerics mode of this implementation."""
    mode: str = "serial"  # serial | parallel
    collapse: int = 2
    threads: int = 1
    kernel_strategy: str = "on_demand"
    scratch_strategy: str = "automatic"
    numerics: str = "fast"  # fast (<=1e-12 rel) | exact (bitwise coal_step) | bott (Bott 1998 flux)

    def to_c(self) -> fsbm_plan:
        for k, table in (("kernel_strategy", _KSTRAT), ("scratch_strategy", _SSTRAT),
                         ("numerics", _NUM)):
            if getattr(self, k) not in table:
                raise ConfigError(f"exec plan: unknown {k} '{getattr(self, k)}'")
        if self.mode not in ("serial", "parallel"):
            raise ConfigError(f"exec plan: unknown mode '{self.mode}'")
        return fsbm_plan(0 if self.mode == "serial" else 1, self.collapse, self.threads,
                         _KSTRAT[self.kernel_strategy], _SSTRAT[self.scratch_strategy],
                         _NUM[self.numerics])


@dataclass
class Ranges:
    """driver.hpp:23-35 (inclusive, 1-based)."""
    ids: int = 1
    ide: int = 1
    kds: int = 1
    kde: int = 1
    jds: int = 1
    jde: int = 1

    def ni(self):
        return self.ide - self.ids + 1

    def nk(self):
        return self.kde - self.kds + 1

    def nj(self):
        return self.jde - self.jds + 1

    def npoints(self):
        return self.ni() * self.nk() * self.nj()

    def to_c(self) -> fsbm_ranges:
        return fsbm_ranges(self.ids, self.ide, self.kds, self.kde, self.jds, self.jde)


@dataclass
class GridState:
    """driver.hpp:40-61: temperature/pressure [npoints], bins[c] [npoints*nkr]
    (point = ((i-ids)*nk + (k-kds))*nj + (j-jds), bin innermost)."""
    ranges: Ranges
    grid: MassGrid
    temperature: object
    pressure: object
    bins: list

    def nkr(self) -> int:
        return self.grid.nkr()

    def point_index(self, i, k, j) -> int:
        r = self.ranges
        return ((i - r.ids) * r.nk() + (k - r.kds)) * r.nj() + (j - r.jds)

    def on_device(self) -> bool:
        return _is_cuda(self.bins[0])


@dataclass
class PredicateMask:
    """driver.hpp:88-95"""
    ranges: Ranges
    call_coal: object
    true_count: int = 0


@dataclass
class PatchTilePlan:
    """driver.hpp:69-80: tiles listed patch-major."""
    tiles: list = field(default_factory=list)  # (its, ite, jts, jte)


def _split_range(lo, hi, parts, what):
    extent = hi - lo + 1
    if parts < 1 or parts > extent:
        raise DomainError(f"decompose: {what} count {parts} does not fit extent {extent}")
    base, rem = divmod(extent, parts)
    out, start = [], lo
    for p in range(parts):
        ln = base + (1 if p < rem else 0)
        out.append((start, start + ln - 1))
        start += ln
    return out


def decompose(ranges: Ranges, n_patches: int, n_tiles_per_patch: int) -> PatchTilePlan:
    """driver.cpp:187-196: j patches, i tiles within each patch."""
    tiles = []
    for jlo, jhi in _split_range(ranges.jds, ranges.jde, n_patches, "patch"):
        for ilo, ihi in _split_range(ranges.ids, ranges.ide, n_tiles_per_patch, "tile"):
            tiles.append((ilo, ihi, jlo, jhi))
    return PatchTilePlan(tiles)


@dataclass
class WorkCounters:
    """CoalCounters (coalescence.hpp:68-71) + KernelTableSet::eval_count."""
    triples: int = 0
    points: int = 0
    kernel_evals: int = 0


@dataclass
class PhaseTimings:
    coal_s: float = 0.0
    step_s: float = 0.0


# ---- device context ------------------------------------------------------------------
def _ptr(a) -> int:
    if a is None:
        return 0
    if _is_cuda(a):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ShapeError("arrays must be C-contiguous")
        return a.ctypes.data
    raise TypeError(f"unsupported array type {type(a)}")


def _is_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


class CoalContext:
    """Owns the device copies of the tables, the registry and the GainTable
    (StepContext{tables, gains}, driver.hpp:141-150)."""

    def __init__(self, grid: MassGrid, tables: KernelTableSet, device: int = 0):
        lib = _lib.load()
        self.grid = grid
        self.tables = tables
        self.nkr = grid.nkr()
        if tables.nkr() != self.nkr:
            raise ShapeError("coal_step: grid, tables and gain table disagree on nkr")
        abd = np.array([[p.source_a, p.source_b, p.dest] for p in tables.pairs], np.int32)
        self._keep = [np.ascontiguousarray(grid.x, np.float64), abd.reshape(-1),
                      np.ascontiguousarray(tables.t750, np.float64).reshape(-1),
                      np.ascontiguousarray(tables.t500, np.float64).reshape(-1)]
        h = C.c_void_p()
        st = lib.fsbm_ctx_create(device, self.nkr, self._keep[0].ctypes.data, grid.ratio,
                                 len(tables.pairs), self._keep[1].ctypes.data,
                                 self._keep[2].ctypes.data, self._keep[3].ctypes.data,
                                 C.byref(h))
        _lib.check(st)
        self.handle = h
        self.device = device

    def fast_kernel(self) -> str:
        """Name of the FSBM_NUMERICS_FAST kernel this context dispatches to."""
        k = C.c_int(0)
        _lib.check(_lib.load().fsbm_ctx_fast_kernel(self.handle, C.byref(k)))
        return {0: "unsupported", 1: "coal_fast", 2: "coal_dmma", 3: "coal_dmmag"}[k.value]

    def gain_table(self):
        """(lo, w_lo, w_hi, top), each [nkr*nkr] -- GainTable::at(i, j) at [i*nkr + j]."""
        n = self.nkr * self.nkr
        lo = np.zeros(n, np.int32)
        wlo, whi, top = np.zeros(n), np.zeros(n), np.zeros(n)
        _lib.check(_lib.load().fsbm_ctx_gain_table(self.handle, lo.ctypes.data, wlo.ctypes.data,
                                                   whi.ctypes.data, top.ctypes.data))
        return lo, wlo, whi, top

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().fsbm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class StepContext:
    """driver.hpp:141-150 (stubs/arena are accepted but have no device meaning)."""
    ctx: CoalContext
    coal: CoalConfig = field(default_factory=CoalConfig)
    counters: Optional[WorkCounters] = None
    timings: Optional[PhaseTimings] = None
    tiles: Optional[PatchTilePlan] = None
    stream: Optional[int] = None


def fission_predicates(state: GridState, ctx: Optional[CoalContext] = None) -> PredicateMask:
    """driver.cpp:198-211. Device state -> computed on device; host state -> host."""
    if state.on_device():
        import torch
        if ctx is None:
            raise DomainError("fission_predicates: device state needs a CoalContext")
        mask = torch.empty(state.ranges.npoints(), dtype=torch.uint8, device=state.bins[0].device)
        cnt = C.c_uint64()
        stream = torch.cuda.current_stream(state.bins[0].device).cuda_stream
        _lib.check(_lib.load().fsbm_fission_predicates_device(
            ctx.handle, state.ranges.npoints(), _ptr(state.temperature), _ptr(mask),
            C.byref(cnt), stream))
        return PredicateMask(state.ranges, mask, int(cnt.value))
    T = np.asarray(state.temperature)
    on = (T > OUTER_GATE_K) & (T > COAL_GATE_K)
    return PredicateMask(state.ranges, on.astype(np.uint8), int(on.sum()))


def _check_buffers(state: GridState, mask: Optional[PredicateMask], ctx: CoalContext) -> None:
    """The C ABI trusts npoints*nkr doubles per category: check dtype, size, contiguity
    and placement of every buffer before handing raw pointers over (ShapeError /
    DomainError, as the reference's GridState/PredicateMask checks, driver.cpp:127-129)."""
    np_ = state.ranges.npoints()
    dev = state.on_device()

    def check(a, name, dtype, n):
        if a is None:
            return
        if _is_cuda(a) != dev:
            raise DomainError(f"fissioned_step: {name} is {'host' if dev else 'device'} memory "
                              f"but the state is on the {'device' if dev else 'host'}")
        if dev:
            import torch
            tdt = {np.float64: torch.float64, np.uint8: torch.uint8}[dtype]
            if a.dtype != tdt:
                raise ShapeError(f"fissioned_step: {name} must be {tdt}, got {a.dtype}")
            if not a.is_contiguous():
                raise ShapeError(f"fissioned_step: {name} must be contiguous")
            if a.device.index != ctx.device:
                raise DomainError(f"fissioned_step: {name} is on cuda:{a.device.index}, "
                                  f"the context on cuda:{ctx.device}")
            size = a.numel()
        else:
            if not isinstance(a, np.ndarray):
                raise ShapeError(f"fissioned_step: {name} must be a numpy array")
            if a.dtype != dtype:
                raise ShapeError(f"fissioned_step: {name} must be {np.dtype(dtype)}, got {a.dtype}")
            if not a.flags.c_contiguous:
                raise ShapeError(f"fissioned_step: {name} must be C-contiguous")
            size = a.size
        if size != n:
            raise ShapeError(f"fissioned_step: {name} has {size} elements, expected {n}")

    if len(state.bins) != NCAT:
        raise ShapeError(f"fissioned_step: state needs {NCAT} category arrays")
    for c, b in enumerate(state.bins):
        if b is None:
            raise DomainError("fissioned_step: null category array")
        check(b, f"bins[{CATEGORIES[c]}]", np.float64, np_ * state.nkr())
    if state.pressure is None:
        raise DomainError("fissioned_step: pressure is required")
    check(state.pressure, "pressure", np.float64, np_)
    check(state.temperature, "temperature", np.float64, np_)
    if mask is not None:
        check(mask.call_coal, "mask", np.uint8, np_)


def fissioned_step(state: GridState, mask: Optional[PredicateMask], step: StepContext,
                   plan: ExecPlan = ExecPlan()) -> None:
    """fissioned_step (driver.hpp:179-180, driver.cpp:353-434) -- phase 2 on the GPU.

    Raises ConfigError / ShapeError / DomainError / StiffnessError (with the
    first failing point in serial order) exactly where the reference throws."""
    import time

    lib = _lib.load()
    ctx = step.ctx
    if mask is not None and mask.ranges != state.ranges:
        raise ShapeError("fissioned_step: mask extents do not match the state")
    if state.nkr() != ctx.nkr:
        raise ShapeError("coal_step: state distribution size does not match nkr")
    _check_buffers(state, mask, ctx)
    cplan = plan.to_c()
    tiles = step.tiles.tiles if step.tiles is not None else []
    tarr = (fsbm_tile * max(1, len(tiles)))(*[fsbm_tile(*t) for t in tiles])
    cnt, err = fsbm_counters(), fsbm_error()
    binsp = (C.c_void_p * NCAT)(*[_ptr(b) for b in state.bins])
    t0 = time.perf_counter()
    if state.on_device():
        import torch
        stream = step.stream
        if stream is None:
            stream = torch.cuda.current_stream(state.bins[0].device).cuda_stream
        st = lib.fsbm_step_grid_device(
            ctx.handle, state.ranges.to_c(), binsp, _ptr(state.pressure),
            _ptr(state.temperature), _ptr(mask.call_coal) if mask is not None else 0,
            step.coal.dt, step.coal.substeps, C.byref(cplan), tarr if tiles else None,
            len(tiles), stream, C.byref(cnt), C.byref(err))
    else:
        st = lib.fsbm_step_grid_host(
            ctx.handle, state.ranges.to_c(), binsp, _ptr(state.pressure),
            _ptr(state.temperature), _ptr(mask.call_coal) if mask is not None else 0,
            step.coal.dt, step.coal.substeps, C.byref(cplan), tarr if tiles else None,
            len(tiles), C.byref(cnt), C.byref(err))
    dt = time.perf_counter() - t0
    if step.timings is not None:
        step.timings.coal_s += dt
        step.timings.step_s += dt
    if step.counters is not None and st in (0, 4):
        step.counters.triples += cnt.triples
        step.counters.points += cnt.points
        step.counters.kernel_evals += cnt.kernel_evals
    _lib.check(st, err)


def coal_step(ctx: CoalContext, n: np.ndarray, pressure: float, cfg: CoalConfig = CoalConfig(),
              numerics: str = "fast", counters: Optional[WorkCounters] = None) -> None:
    """coal_step (coalescence.hpp:148-150) on one point: n is (6, nkr) float64, in place."""
    if n.shape != (NCAT, ctx.nkr) or n.dtype != np.float64 or not n.flags.c_contiguous:
        raise ShapeError("coal_step: state distribution size does not match nkr")
    if cfg.kernel_strategy not in _KSTRAT or numerics not in _NUM:
        raise ConfigError("coal_step: unknown strategy")
    cnt, err = fsbm_counters(), fsbm_error()
    st = _lib.load().fsbm_coal_step(ctx.handle, n.ctypes.data, pressure, cfg.dt, cfg.substeps,
                                    _KSTRAT[cfg.kernel_strategy], _NUM[numerics], C.byref(cnt),
                                    C.byref(err))
    if counters is not None and st == 0:
        counters.triples += cnt.triples
        counters.points += cnt.points
        counters.kernel_evals += cnt.kernel_evals
    _lib.check(st, err)
