"""GPU parity of FSBM_NUMERICS_BOTT (Bott 1998 flux method, csrc/coal_bott.cuh) against its
oracle (oracle/bott_oracle.c, pinned by tests/test_oracle_bott.py), through the C ABI.

Bar: counters bit-exact; bins per value |gpu - ref| <= RTOL |ref| + ATOL_FRAC sum_k ref_c[k]
(the kernel rounds every product/sum like the oracle; only libdevice log/log1p/exp/expm1
differ from glibc's by an ulp or two, so the sequential sweep stays within round-off);
mass conserved per point to 1e-13; never negative, even where Kovetz-Olund is stiff;
host path == device path and run-to-run bitwise."""
import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm

from test_gpu_parity import device_state, make_ctx, oracle_inputs, thunder_host

pytestmark = pytest.mark.gpu

RTOL = 1e-12
ATOL_FRAC = 1e-15


def bott_oracle(oracle, ctx, tabs, st, mask, B, dt=1.0, substeps=1, kstrat=1):
    x, abd, t750, t500, g = oracle_inputs(oracle, ctx, tabs)
    cour = oracle.bott_courant(x, g[0])
    Bo = np.ascontiguousarray(B.copy())
    s, cnt = oracle.bott_step_grid(x, abd, t750, t500, g[0], cour, mask, np.asarray(st.pressure), Bo,
                                   dt, substeps, kstrat)
    assert s == 0
    return cnt, Bo


def close(got, ref, point_floor=False):
    """Out-of-tolerance count and worst relative error.  point_floor: the absolute floor scales
    with the point's total number over all categories (a category the step nearly empties
    keeps an absolute error at that scale, not at its own vanishing total)."""
    scale = np.abs(ref).sum(axis=-1, keepdims=True)
    if point_floor:
        scale = np.broadcast_to(np.abs(ref).sum(axis=(0, 2), keepdims=True), scale.shape)
    err = np.abs(got - ref) - (RTOL * np.abs(ref) + ATOL_FRAC * scale)
    return int((err > 0).sum()), float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)))


def step_device(ctx, st, mask, substeps=1, kstrat="on_demand", dt=1.0):
    d = device_state(st)
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(d, mask, fsbm.StepContext(ctx, coal=fsbm.CoalConfig(dt, substeps), counters=cnt),
                        fsbm.ExecPlan(kernel_strategy=kstrat, numerics="bott"))
    return np.stack([b.cpu().numpy().reshape(-1, ctx.nkr) for b in d.bins]), cnt


@pytest.mark.parametrize("nkr,dims", [(17, (3, 8, 20)), (33, (3, 10, 40)), (66, (2, 4, 12)),
                                      (132, (1, 3, 6)), (264, (1, 2, 3))])
def test_bott_grid_vs_oracle(oracle, nkr, dims):
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, *dims, 0.9, 42)
    cnt_o, Bo = bott_oracle(oracle, ctx, tabs, st, mask, B)
    got, cnt = step_device(ctx, st, None)
    bad, worst = close(got, Bo)
    assert bad == 0, (bad, worst)
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
    m = ~mask.astype(bool)  # mask-false points untouched, bitwise
    assert np.array_equal(got[:, m], B[:, m])


@pytest.mark.parametrize("substeps,kstrat", [(3, "on_demand"), (2, "precomputed")])
def test_bott_substeps_and_counters(oracle, substeps, kstrat):
    nkr = 33
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, 2, 6, 20, 0.7, 7)
    cnt_o, Bo = bott_oracle(oracle, ctx, tabs, st, mask, B, substeps=substeps,
                            kstrat=0 if kstrat == "precomputed" else 1)
    got, cnt = step_device(ctx, st, None, substeps=substeps, kstrat=kstrat)
    bad, worst = close(got, Bo)
    assert bad == 0, (bad, worst)
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]


def test_bott_positive_where_kovetz_olund_is_stiff(oracle):
    """coeff 1500 at dt = 1 makes coal_step throw StiffnessError (SURVEY 8(d) probe); Bott's
    limiters keep every bin >= 0 and conserve each point's mass."""
    nkr = 33
    ctx, grid, tabs = make_ctx(nkr, coeff=1500.0)
    st, mask, B = thunder_host(oracle, ctx, 2, 5, 16, 1.0, 11)
    with pytest.raises(fsbm.StiffnessError):
        fsbm.fissioned_step(device_state(st), None, fsbm.StepContext(ctx), fsbm.ExecPlan())
    cnt_o, Bo = bott_oracle(oracle, ctx, tabs, st, mask, B)
    got, _ = step_device(ctx, st, None)
    assert (got >= 0.0).all()
    x = grid.x
    m0, m1 = (B * x).sum(axis=(0, 2)), (got * x).sum(axis=(0, 2))
    np.testing.assert_allclose(m1, m0, rtol=1e-13)
    bad, worst = close(got, Bo, point_floor=True)
    assert bad == 0, (bad, worst)


def test_bott_host_equals_device_and_deterministic(oracle):
    nkr = 33
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, 3, 6, 30, 0.8, 5)
    d1, _ = step_device(ctx, st, None)
    d2, _ = step_device(ctx, st, None)
    assert np.array_equal(d1, d2)
    h = fsbm.GridState(st.ranges, grid, st.temperature.copy(), st.pressure.copy(),
                       [b.copy() for b in st.bins])
    fsbm.fissioned_step(h, None, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics="bott"))
    assert np.array_equal(np.stack([b.reshape(-1, nkr) for b in h.bins]), d1)


def test_bott_multistep_mass_and_number():
    """20 Bott steps of the thunderstorm state: domain mass constant to round-off, number
    non-increasing (collisions only merge particles)."""
    import torch
    from paper_2409_07232_b200 import synth
    nkr = 33
    ctx, grid, tabs = make_ctx(nkr)
    st, mask = synth.thunderstorm_device(ctx, 4, 10, 50, 1.0, 3)
    x = torch.tensor(grid.x, device="cuda:0")
    mass = lambda: sum(float((b.view(-1, nkr) * x).sum()) for b in st.bins)
    number = lambda: sum(float(b.sum()) for b in st.bins)
    m0, n_prev = mass(), number()
    for _ in range(20):
        fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics="bott"))
        n = number()
        assert n <= n_prev * (1 + 1e-14)
        n_prev = n
    assert abs(mass() - m0) <= 1e-12 * m0
    assert all(float(b.min()) >= 0.0 for b in st.bins)
