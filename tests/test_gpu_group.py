"""Multi-GPU path on one B200: a device group with two contexts on cuda:0 (fsbm_group_*),
i-slab and WRF j-patch shards, against one context and against the oracle.

Results are bitwise independent of the decomposition: EXACT always; FAST
because the batched kernels group points within one model level (level-major compaction),
so with pressure constant on a level -- the reference's synthetic profile -- every group has
one weight and a point's arithmetic never depends on its batch partners.  Counters, the
first failing point and the diagnostics are whole-domain."""
import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm
from paper_2409_07232_b200 import shard, synth

pytestmark = pytest.mark.gpu

from test_gpu_parity import assert_close, make_ctx, run_oracle_grid, thunder_host  # noqa: E402


def group_for(grid, tabs, devices=(0, 0)):
    return fsbm.DeviceGroup(grid, tabs, list(devices))


def host_copy(st):
    return fsbm.GridState(st.ranges, st.grid, st.temperature.copy(), st.pressure.copy(),
                          [b.copy() for b in st.bins])


@pytest.mark.parametrize("split", ["i", "j"])
@pytest.mark.parametrize("numerics", ["exact", "fast"])
@pytest.mark.parametrize("nkr", [33, 66])
def test_group_host_two_contexts_equal_one(oracle, split, numerics, nkr):
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, 6, 5, 9, 0.8, 42)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 0
    one = host_copy(st)
    plan = fsbm.ExecPlan(numerics=numerics)
    fsbm.fissioned_step(one, None, fsbm.StepContext(ctx), plan)
    g = group_for(grid, tabs)
    two = host_copy(st)
    cnt = fsbm.WorkCounters()
    g.step_host(two, None, split, plan=plan, counters=cnt)
    got = np.stack([b.reshape(-1, nkr) for b in two.bins])
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
    if numerics == "exact":
        assert np.array_equal(got, Bo)
    else:
        assert_close(got, Bo, f"group {split}")
    assert np.array_equal(got, np.stack([b.reshape(-1, nkr) for b in one.bins]))
    off = mask == 0
    assert np.array_equal(got[:, off], B[:, off])


@pytest.mark.parametrize("split", ["i", "j"])
def test_group_device_shards_and_diagnostics(oracle, split):
    """Device-resident shards (each its own arrays, global ranges) + NCCL-free reduction:
    counters and number/mass diagnostics are the whole domain's."""
    import torch
    ctx, grid, tabs = make_ctx(33)
    st, mask, B = thunder_host(oracle, ctx, 5, 4, 8, 1.0, 7)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    full = st.ranges
    parts = shard.decompose_shards(full, 2, split)
    dev = torch.device("cuda:0")
    states = []
    for r in parts:
        i = np.arange(r.ids - 1, r.ide)[:, None, None]
        k = np.arange(full.nk())[None, :, None]
        j = np.arange(r.jds - 1, r.jde)[None, None, :]
        idx = ((i * full.nk() + k) * full.nj() + j).reshape(-1)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        states.append((idx, fsbm.GridState(r, grid, t(st.temperature[idx]), t(st.pressure[idx]),
                                           [t(B[c, idx].reshape(-1)) for c in range(6)])))
    g = group_for(grid, tabs)
    cnt = fsbm.WorkCounters()
    diag = g.step_device([s_ for _, s_ in states], [None, None], plan=fsbm.ExecPlan(numerics="exact"),
                         counters=cnt, diagnostics=True)
    got = np.zeros_like(Bo)
    for idx, s_ in states:
        got[:, idx] = np.stack([b.cpu().numpy().reshape(-1, 33) for b in s_.bins])
    assert np.array_equal(got, Bo)
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
    np.testing.assert_allclose(diag.number_before, B.sum(axis=(1, 2)), rtol=1e-13)
    np.testing.assert_allclose(diag.mass_after, (Bo * grid.x).sum(axis=(1, 2)), rtol=1e-13)
    assert abs(diag.mass_after.sum() - diag.mass_before.sum()) <= 1e-12 * diag.mass_before.sum()
    assert diag.coal_kernel_ms_max > 0


def test_group_stiffness_reports_the_serial_first_point(oracle):
    """Stiffness in several shards: the group reports the point the serial reference
    would, first in (tile, j, k, i) order over the WHOLE domain."""
    ctx, grid, tabs = make_ctx(33, coeff=1500.0)
    st, mask, B = thunder_host(oracle, ctx, 4, 2, 6, 1.0, 5)
    tiles = fsbm.decompose(st.ranges, 2, 2)
    from test_gpu_parity import oracle_inputs
    x, abd, t750, t500, gt = oracle_inputs(oracle, ctx, tabs)
    want = None
    for (its, ite, jts, jte) in tiles.tiles:
        for j in range(jts, jte + 1):
            for k in range(1, st.ranges.nk() + 1):
                for i in range(its, ite + 1):
                    p = st.point_index(i, k, j)
                    if want is None and mask[p]:
                        b = np.ascontiguousarray(B[:, p])
                        s, _, ce = oracle.coal_step(x, abd, t750, t500, gt, b, float(st.pressure[p]))
                        if s == 4:
                            want = ((i, k, j), ce)
    assert want is not None
    g = group_for(grid, tabs)
    for split in ("i", "j"):
        with pytest.raises(fsbm.StiffnessError) as ei:
            g.step_host(host_copy(st), None, split, tiles=tiles, plan=fsbm.ExecPlan(numerics="exact"))
        assert ei.value.point == want[0]
        assert (ei.value.category, ei.value.bin) == want[1]
        assert ei.value.value < 0 and "would become negative (" in str(ei.value)


def test_group_stale_mask_and_config_errors(oracle):
    ctx, grid, tabs = make_ctx(33)
    st, mask, B = thunder_host(oracle, ctx, 4, 3, 4, 0.5, 3)
    g = group_for(grid, tabs)
    bad = fsbm.PredicateMask(st.ranges, mask.astype(np.uint8).copy())
    bad.call_coal[-1] ^= 1  # a point in the LAST shard only
    with pytest.raises(fsbm.DomainError, match="stale"):
        g.step_host(host_copy(st), bad, "j")
    with pytest.raises(fsbm.ConfigError):
        g.step_host(host_copy(st), None, "i", plan=fsbm.ExecPlan("parallel", 3, 1, "on_demand",
                                                                 "automatic"))
    with pytest.raises(fsbm.DomainError):  # more shards than j columns
        fsbm.DeviceGroup(grid, tabs, [0] * 5).step_host(host_copy(st), None, "j")


@pytest.mark.parametrize("cf", [0.05, 0.3])
@pytest.mark.parametrize("nkr", [33, 66])
def test_group_sparse_masks_bitwise(oracle, cf, nkr):
    """Sparse scattered masks (most 16-point groups of the level-major list carry holes, many
    levels hold fewer than 16 active points): counters exact, FAST within the bar, and the
    j-patch group bitwise equal to one context."""
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, 7, 6, 11, cf, 3)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 0
    one = host_copy(st)
    c1 = fsbm.WorkCounters()
    fsbm.fissioned_step(one, None, fsbm.StepContext(ctx, counters=c1), fsbm.ExecPlan())
    got1 = np.stack([b.reshape(-1, nkr) for b in one.bins])
    assert [c1.triples, c1.points, c1.kernel_evals] == [int(v) for v in cnt_o]
    assert_close(got1, Bo, f"sparse cf {cf}")
    g = group_for(grid, tabs, (0, 0, 0))
    two = host_copy(st)
    g.step_host(two, None, "j")
    assert np.array_equal(np.stack([b.reshape(-1, nkr) for b in two.bins]), got1)
