"""Multi-GPU sharding of the coalescence step (host side).

Microphysics is column-local: coal_step touches only its own point,
so the domain shards into independent i-slabs with no halo and no data-path
collective.  i is the slowest index of GridState::point_index (driver.hpp:49-53),
so a slab is one contiguous range of every per-category array.  The only
collective is the end-of-step diagnostic reduction (counters, mass before/after,
first failing point), one small all-reduce per step.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def decompose_shards(ranges, nshards: int, split: str = "i") -> list:
    """fsbm_decompose (C ABI; split_range, driver.cpp:35-51): nshards near-equal i-slabs
    ("i") or WRF j-patches ("j", decompose, driver.cpp:187-196) of `ranges`, all k."""
    import ctypes as C

    from . import _lib
    from .coalbench import Ranges
    out = (_lib.fsbm_ranges * max(1, nshards))()
    _lib.check(_lib.load().fsbm_decompose(ranges.to_c(), nshards, {"i": 0, "j": 1}[split], out))
    return [Ranges(o.ids, o.ide, o.kds, o.kde, o.jds, o.jde) for o in out[:nshards]]


def slab(ni: int, world: int, rank: int) -> tuple[int, int]:
    """Rank's i-slab of [0, ni) (sizes differ by <= 1, remainder to the first ranks), from
    fsbm_decompose.  Returns (i0, i1), 0-based half-open."""
    from .coalbench import Ranges
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if ni < world:
        raise ValueError(f"cannot split {ni} i-rows over {world} ranks")
    r = decompose_shards(Ranges(1, ni, 1, 1, 1, 1), world, "i")[rank]
    return r.ids - 1, r.ide


def shard_slice(ni: int, nk: int, nj: int, world: int, rank: int) -> tuple[int, int]:
    """Point range [p0, p1) of this rank's slab in the global (i,k,j) numbering."""
    i0, i1 = slab(ni, world, rank)
    return i0 * nk * nj, i1 * nk * nj


@dataclass
class StepDiagnostics:
    """Per-step diagnostics; the only data crossing ranks."""
    triples: int = 0
    points: int = 0
    kernel_evals: int = 0
    mass_before: float = 0.0
    mass_after: float = 0.0
    number_before: float = 0.0
    number_after: float = 0.0
    first_error_key: int = -1  # global serial-order key of the first failing point, -1 none

    def pack(self):
        ints = np.array([self.triples, self.points, self.kernel_evals,
                         self.first_error_key if self.first_error_key >= 0 else np.iinfo(np.int64).max],
                        dtype=np.int64)
        flts = np.array([self.mass_before, self.mass_after, self.number_before,
                         self.number_after], dtype=np.float64)
        return ints, flts

    @staticmethod
    def unpack(ints, flts) -> "StepDiagnostics":
        key = int(ints[3])
        return StepDiagnostics(int(ints[0]), int(ints[1]), int(ints[2]), float(flts[0]),
                               float(flts[1]), float(flts[2]), float(flts[3]),
                               -1 if key == np.iinfo(np.int64).max else key)


def reduce_diagnostics(d: StepDiagnostics, dist=None, device=None) -> StepDiagnostics:
    """All-reduce over the process group (NCCL on GPUs, gloo on CPU): counters and
    masses summed, first failing point = min key.  No-op without a process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return d
    import torch
    ints, flts = d.pack()
    ti = torch.from_numpy(ints[:3].copy()).to(device or "cpu")
    tk = torch.from_numpy(ints[3:].copy()).to(device or "cpu")
    tf = torch.from_numpy(flts.copy()).to(device or "cpu")
    dist.all_reduce(ti, op=dist.ReduceOp.SUM)
    dist.all_reduce(tk, op=dist.ReduceOp.MIN)
    dist.all_reduce(tf, op=dist.ReduceOp.SUM)
    return StepDiagnostics.unpack(np.concatenate([ti.cpu().numpy(), tk.cpu().numpy()]),
                                  tf.cpu().numpy())
