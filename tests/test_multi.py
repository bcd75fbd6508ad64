"""N>1 path on CPU: world_size-2 gloo process group, the product's shard plan
(fsbm_decompose: i-slabs and WRF j-patches), the oracle as the per-shard step (no GPU
here), diagnostics all-reduced by shard.reduce_diagnostics; the merged state must equal
the single-process step bitwise and the diagnostics must match.  The device path of the
same plan (fsbm_group_step_*) is tested on the GPU in tests/test_gpu_group.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_07232_b200 import shard

NI, NK, NJ, NKR, SEED = 5, 3, 4, 33, 42


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(oracle):
    import paper_2409_07232_b200 as fsbm
    from paper_2409_07232_b200 import synth
    grid = fsbm.make_mass_grid(NKR)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(), fsbm.KernelParams("golovin", 1, 1.5, 0.05))
    T, P, _ = synth.thermo_host(NI, NK, NJ, 0.8, SEED, grid)
    mask, _ = oracle.fission_predicates(T)
    B = oracle.thunderstorm_block(grid.x, SEED, 0, NI * NK * NJ, mask)
    return grid, tabs, T, P, mask, B


def _shard_index(r):
    """Flat indices (reference layout of the full grid) of shard r's points, in the
    reference layout of the shard itself."""
    i = np.arange(r.ids - 1, r.ide)[:, None, None]
    k = np.arange(NK)[None, :, None]
    j = np.arange(r.jds - 1, r.jde)[None, None, :]
    return ((i * NK + k) * NJ + j).reshape(-1)


def _run_shard(oracle, grid, tabs, P, mask, B, r):
    idx = _shard_index(r)
    Bs = np.ascontiguousarray(B[:, idx])
    abd = oracle.default_registry()
    g = oracle.gain_table(grid.x, grid.ratio)
    x = grid.x
    m0 = float((Bs * x).sum())
    st, cnt, err = oracle.step_grid(r.ni(), NK, r.nj(), x, abd, tabs.t750.reshape(-1).copy(),
                                    tabs.t500.reshape(-1).copy(), g,
                                    np.ascontiguousarray(mask[idx]), np.ascontiguousarray(P[idx]), Bs)
    assert st == 0
    d = shard.StepDiagnostics(int(cnt[0]), int(cnt[1]), int(cnt[2]), m0, float((Bs * x).sum()),
                              0.0, 0.0, -1)
    return Bs, d


def _worker(rank, world, port, out, split):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pyoracle
    from paper_2409_07232_b200 import Ranges
    O = pyoracle.Oracle()
    grid, tabs, T, P, mask, B = _problem(O)
    r = shard.decompose_shards(Ranges(1, NI, 1, NK, 1, NJ), world, split)[rank]
    Bs, d = _run_shard(O, grid, tabs, P, mask, B, r)
    tot = shard.reduce_diagnostics(d, dist)
    np.save(os.path.join(out, f"shard{rank}.npy"), Bs)
    if rank == 0:
        np.save(os.path.join(out, "diag.npy"), np.array([tot.triples, tot.points, tot.kernel_evals,
                                                         tot.mass_before, tot.mass_after]))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_partition():
    assert shard.slab(425, 8, 0) == (0, 54) and shard.slab(425, 8, 7) == (372, 425)
    for world in (1, 2, 3, 4, 8):
        spans = [shard.slab(425, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 425
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard.slab(3, 4, 0)


@pytest.mark.parametrize("split", ["i", "j"])
def test_two_rank_gloo_equals_single(tmp_path, oracle, split):
    from paper_2409_07232_b200 import Ranges
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), split), nprocs=world, join=True)
    grid, tabs, T, P, mask, B = _problem(oracle)
    full = Ranges(1, NI, 1, NK, 1, NJ)
    Bfull, dfull = _run_shard(oracle, grid, tabs, P, mask, B, full)
    merged = np.zeros_like(Bfull)
    for rk, r in enumerate(shard.decompose_shards(full, world, split)):
        merged[:, _shard_index(r)] = np.load(tmp_path / f"shard{rk}.npy")
    assert np.array_equal(merged, Bfull)  # sharding never changes a point's result
    diag = np.load(tmp_path / "diag.npy")
    assert list(diag[:3].astype(np.int64)) == [dfull.triples, dfull.points, dfull.kernel_evals]
    assert abs(diag[3] - dfull.mass_before) <= 1e-13 * dfull.mass_before
    assert abs(diag[4] - dfull.mass_after) <= 1e-13 * dfull.mass_after
