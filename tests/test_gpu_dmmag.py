"""GPU parity of coal_dmmag (the general-band FP64 tensor-core kernel) against the oracle.

Forced with FSBM_FAST_KERNEL=dmmag at context creation so it also runs on the grids
the tuned 33-bin kernel normally takes; the default dispatch at 17/66 bins selects it
by itself (checked).  Same bar as test_gpu_parity.py: per bin
|gpu - ref| <= 1e-12 |ref| + 1e-15 sum_k ref_c[k], counters exact, mask-false points
bit-identical.
"""
import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm
from test_gpu_parity import assert_close, device_state, make_ctx, run_oracle_grid, thunder_host

pytestmark = pytest.mark.gpu


@pytest.fixture
def forced(monkeypatch):
    monkeypatch.setenv("FSBM_FAST_KERNEL", "dmmag")


@pytest.mark.parametrize("nkr", [17, 66, 132, 264])
def test_default_dispatch_picks_dmmag(nkr):
    ctx, _, _ = make_ctx(nkr)
    assert ctx.fast_kernel() == "coal_dmmag"


@pytest.mark.parametrize("nkr,ratio,pmode,dims", [
    (33, None, "levels", (4, 5, 37)),
    (33, None, "random", (3, 4, 29)),
    (17, None, "levels", (5, 4, 21)),
    (20, 1.7, "random", (3, 5, 19)),   # non-doubling grid, 3-row tail block
    (66, None, "levels", (2, 5, 33)),
    (66, None, "random", (2, 3, 21)),
    (48, 1.35, "levels", (2, 4, 17)),  # wider band (targets up to o+5)
    (90, None, "levels", (1, 3, 17)),  # 12 blocks: 16-point batches (shared-memory fit)
    (132, None, "levels", (1, 2, 19)), # 17 blocks, targets up to o+5
    (132, None, "random", (1, 2, 13)),
    (264, None, "levels", (1, 1, 21)), # 33 blocks, targets up to o+9, lean shared-memory layout
    (200, None, "random", (1, 1, 9)),
])
def test_dmmag_vs_oracle(oracle, forced, nkr, ratio, pmode, dims):
    ctx, grid, tabs = make_ctx(nkr, ratio=ratio)
    assert ctx.fast_kernel() == "coal_dmmag"
    st, mask, B = thunder_host(oracle, ctx, *dims, 0.8, 7)
    if pmode == "random":
        rng = np.random.default_rng(3)
        st.pressure[:] = rng.uniform(350.0, 950.0, st.pressure.shape)
        st.pressure[::5] = 640.0
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=0.5)
    assert s == 0
    dst = device_state(st)
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(dst, None, fsbm.StepContext(ctx, fsbm.CoalConfig(0.5, 1), cnt), fsbm.ExecPlan())
    got = np.stack([b.cpu().numpy().reshape(-1, nkr) for b in dst.bins])
    assert_close(got, Bo, f"dmmag nkr{nkr} ratio{ratio} {pmode}")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
    off = mask == 0
    assert np.array_equal(got[:, off], B[:, off])


@pytest.mark.parametrize("nkr", [33, 66])
def test_dmmag_substeps_precomputed(oracle, forced, nkr):
    ctx, grid, tabs = make_ctx(nkr)
    st, mask, B = thunder_host(oracle, ctx, 2, 3, 11, 1.0, 9)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=1.5, substeps=3, kstrat=0)
    assert s == 0
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, fsbm.CoalConfig(1.5, 3), cnt),
                        fsbm.ExecPlan(kernel_strategy="precomputed"))
    got = np.stack([b.reshape(-1, nkr) for b in st.bins])
    assert_close(got, Bo, "dmmag substeps")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]


def test_dmmag_deterministic_and_conserving(oracle, forced):
    ctx, grid, tabs = make_ctx(66)
    st, mask, B = thunder_host(oracle, ctx, 2, 4, 23, 0.9, 17)
    outs = []
    for _ in range(2):
        d = device_state(st)
        fsbm.fissioned_step(d, None, fsbm.StepContext(ctx), fsbm.ExecPlan())
        outs.append(np.stack([b.cpu().numpy().reshape(-1, 66) for b in d.bins]))
    assert np.array_equal(outs[0], outs[1])
    m0 = (B * grid.x).sum(axis=(0, 2))
    m1 = (outs[0] * grid.x).sum(axis=(0, 2))
    assert np.all(np.abs(m1 - m0) <= 1e-12 * np.maximum(m0, 1e-300))


def test_dmmag_stiffness_first_point(oracle, forced):
    ctx, grid, tabs = make_ctx(66, coeff=1500.0)
    st, mask, B = thunder_host(oracle, ctx, 2, 3, 9, 1.0, 5)
    s, _, err_o, _ = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s != 0
    with pytest.raises(fsbm.StiffnessError) as ei:
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), fsbm.ExecPlan())
    e = ei.value
    assert e.point == tuple(int(v) for v in err_o[2:5])
    assert (e.category, e.bin) == (int(err_o[0]), int(err_o[1]))


@pytest.mark.parametrize("nkr", [33, 66])
def test_dmmag_custom_registry_aliasing(oracle, forced, nkr):
    """Non-standard registry through coal_dmmag: a==dest cross pair, 3-category pair,
    repeated dest, a pair whose source_b is another pair's dest."""
    pairs = [fsbm.InteractionPair("gl", 5, 0, 5), fsbm.InteractionPair("sl", 4, 0, 5),
             fsbm.InteractionPair("ll", 0, 0, 0), fsbm.InteractionPair("il", 1, 0, 0),
             fsbm.InteractionPair("sg", 4, 5, 5)]
    ctx, grid, tabs = make_ctx(nkr, pairs=pairs, coeff=0.05)
    assert ctx.fast_kernel() == "coal_dmmag"
    st, mask, B = thunder_host(oracle, ctx, 2, 3, 7, 1.0, 9)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=0.2)
    assert s == 0
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, fsbm.CoalConfig(0.2), cnt), fsbm.ExecPlan())
    got = np.stack([b.reshape(-1, nkr) for b in st.bins])
    assert_close(got, Bo, f"dmmag custom registry nkr{nkr}")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
