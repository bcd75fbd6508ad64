"""GPU parity: the sm_100a kernels (through the C ABI) against the oracle.

Bar: flux-target selection, masks, counters, stiffness points -> bit-exact;
FSBM_NUMERICS_EXACT -> bitwise equal to coal_step; FSBM_NUMERICS_FAST -> per bin
|gpu - ref| <= RTOL*|ref| + ATOL_FRAC*sum_k ref_c[k] (RTOL = 1e-12, ATOL_FRAC = 1e-15,
north_star: "tighter if the reference is FP64"), mass conserved per point to 1e-12.
"""
import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm
from paper_2409_07232_b200 import synth

pytestmark = pytest.mark.gpu

RTOL = 1e-12
ATOL_FRAC = 1e-15


def make_ctx(nkr, pair_scale_step=0.05, coeff=1.0, family="golovin", pairs=None, ratio=None):
    r = ratio or fsbm.equal_range_ratio(nkr)
    grid = fsbm.make_mass_grid(nkr, 3.35e-14, r)
    pairs = pairs or fsbm.default_pair_registry()
    tabs = fsbm.build_tables(grid, pairs, fsbm.KernelParams(family, coeff, 1.5, pair_scale_step))
    return fsbm.CoalContext(grid, tabs), grid, tabs


def oracle_inputs(oracle, ctx, tabs):
    x = ctx.grid.x
    abd = np.array([[p.source_a, p.source_b, p.dest] for p in tabs.pairs], np.int32).reshape(-1)
    g = oracle.gain_table(x, ctx.grid.ratio)
    return x, abd, tabs.t750.reshape(-1).copy(), tabs.t500.reshape(-1).copy(), g


def assert_close(got, ref, what=""):
    got = np.asarray(got).reshape(ref.shape)
    scale = np.abs(ref).sum(axis=-1, keepdims=True)
    tol = RTOL * np.abs(ref) + ATOL_FRAC * scale
    bad = np.abs(got - ref) > tol
    assert not bad.any(), f"{what}: {bad.sum()} bins out of tolerance, max rel " \
        f"{np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300))}"


def device_state(state):
    import torch
    dev = torch.device("cuda:0")
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return fsbm.GridState(state.ranges, state.grid, t(state.temperature), t(state.pressure),
                          [t(b) for b in state.bins])


def thunder_host(oracle, ctx, ni, nk, nj, cf, seed):
    T, P, _ = synth.thermo_host(ni, nk, nj, cf, seed, ctx.grid)
    mask, _ = oracle.fission_predicates(T)
    nkr = ctx.nkr
    B = np.zeros((6, ni * nk * nj, nkr))
    for p in np.nonzero(mask)[0]:
        B[:, p, :] = oracle.thunderstorm_point(ctx.grid.x, seed, int(p))
    st = fsbm.GridState(fsbm.Ranges(1, ni, 1, nk, 1, nj), ctx.grid, T, P,
                        [B[c].reshape(-1).copy() for c in range(6)])
    return st, mask, B


def run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=1.0, substeps=1, kstrat=1):
    x, abd, t750, t500, g = oracle_inputs(oracle, ctx, tabs)
    r = st.ranges
    Bo = B.copy()
    s, cnt, err = oracle.step_grid(r.ni(), r.nk(), r.nj(), x, abd, t750, t500, g, mask,
                                   np.asarray(st.pressure), Bo, dt, substeps, kstrat)
    return s, cnt, err, Bo


# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("nkr", [17, 33, 66, 132, 264])
def test_gain_table_bitwise(oracle, nkr):
    ctx, grid, _ = make_ctx(nkr)
    got = ctx.gain_table()
    want = oracle.gain_table(grid.x, grid.ratio)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_spec_hand_oracles(numerics):
    for x, init, want in (([1.0, 2.0], [2.0, 0.0], [1.6, 0.2]),
                          ([1.0, 2.0, 4.0], [0.0, 1.0, 0.0], [0.0, 0.9, 0.05])):
        grid = fsbm.make_mass_grid(len(x), 1.0, 2.0)
        pairs = [fsbm.InteractionPair("cwll", 0, 0, 0)]
        tabs = fsbm.build_tables(grid, pairs, fsbm.KernelParams("constant", 1.0, 1.0))
        ctx = fsbm.CoalContext(grid, tabs)
        n = np.zeros((6, len(x)))
        n[0] = init
        fsbm.coal_step(ctx, n, 600.0, fsbm.CoalConfig(dt=0.1), numerics=numerics)
        np.testing.assert_allclose(n[0], want, rtol=0, atol=1e-15)


@pytest.mark.parametrize("nkr", [17, 33, 66])
@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_golden_points(golden, nkr, numerics):
    ctx, _, _ = make_ctx(nkr)
    pin = golden[f"point_nkr{nkr}_in"]
    for q, pres in enumerate(golden[f"point_nkr{nkr}_pressure"]):
        n = pin[q].copy()
        cnt = fsbm.WorkCounters()
        fsbm.coal_step(ctx, n, float(pres), fsbm.CoalConfig(1.0, 2 if q == 1 else 1),
                       numerics=numerics, counters=cnt)
        ref = golden[f"point_nkr{nkr}_out"][q]
        if numerics == "exact":
            assert np.array_equal(n, ref)
        else:
            assert_close(n, ref, f"nkr{nkr} q{q}")
        assert [cnt.triples, cnt.points, cnt.kernel_evals] == list(golden[f"point_nkr{nkr}_counters"][q])


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_golden_small_grid_liquid(golden, numerics):
    nkr = 33
    ctx, grid, _ = make_ctx(nkr)
    ni, nk, nj = 4, 5, 6
    st = fsbm.GridState(fsbm.Ranges(1, ni, 1, nk, 1, nj), grid, golden["grid_T"].copy(),
                        golden["grid_P"].copy(), [golden["grid_in"][c].reshape(-1).copy() for c in range(6)])
    mask = fsbm.fission_predicates(st)
    cnt = fsbm.WorkCounters()
    plan = fsbm.ExecPlan("parallel", 3, 8, "on_demand", "arena", numerics)
    fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx, counters=cnt), plan)
    got = np.stack([b.reshape(-1, nkr) for b in st.bins])
    ref = golden["grid_out"]
    if numerics == "exact":
        assert np.array_equal(got, ref)
    else:
        assert_close(got, ref, "grid")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == list(golden["grid_counters"])


@pytest.mark.parametrize("nkr", [17, 33, 66, 132, 264])
@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_thunderstorm_grid_vs_oracle(oracle, nkr, numerics):
    ctx, grid, tabs = make_ctx(nkr)
    dims = {17: (5, 4, 6), 33: (6, 5, 7), 66: (3, 4, 5), 132: (2, 3, 3), 264: (1, 2, 3)}[nkr]
    st, mask, B = thunder_host(oracle, ctx, *dims, 0.7, 42)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 0
    dst = device_state(st)
    cnt = fsbm.WorkCounters()
    plan = fsbm.ExecPlan("parallel", 3, 4, "on_demand", "arena", numerics)
    fsbm.fissioned_step(dst, fsbm.PredicateMask(st.ranges, None), fsbm.StepContext(ctx, counters=cnt), plan)
    got = np.stack([b.cpu().numpy().reshape(-1, nkr) for b in dst.bins])
    if numerics == "exact":
        assert np.array_equal(got, Bo)
    else:
        assert_close(got, Bo, f"nkr{nkr}")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]
    # untouched (mask-false) points are bit-identical
    off = mask == 0
    assert np.array_equal(got[:, off], B[:, off])


@pytest.mark.parametrize("numerics", ["exact", "fast"])
@pytest.mark.parametrize("substeps,kstrat", [(4, "on_demand"), (2, "precomputed")])
def test_substeps_and_strategies(oracle, numerics, substeps, kstrat):
    ctx, grid, tabs = make_ctx(33)
    st, mask, B = thunder_host(oracle, ctx, 3, 4, 5, 1.0, 3)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=1.5, substeps=substeps,
                                      kstrat=0 if kstrat == "precomputed" else 1)
    assert s == 0
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, fsbm.CoalConfig(1.5, substeps), cnt),
                        fsbm.ExecPlan(kernel_strategy=kstrat, numerics=numerics))
    got = np.stack([b.reshape(-1, 33) for b in st.bins])
    if numerics == "exact":
        assert np.array_equal(got, Bo)
    else:
        assert_close(got, Bo, "substeps")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]


def test_liquid_only_c1_fast(oracle):
    """C1: the reference's own make_synthetic_case 32x40x32, 33 bins (only cwll active)."""
    ctx, grid, tabs = make_ctx(33)
    st = synth.liquid_case_host(32, 40, 32, 1.0, 42, grid)
    B = np.stack([b.reshape(-1, 33) for b in st.bins]).copy()
    mask, _ = oracle.fission_predicates(st.temperature)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 0
    dst = device_state(st)
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(dst, None, fsbm.StepContext(ctx, counters=cnt), fsbm.ExecPlan())
    got = np.stack([b.cpu().numpy().reshape(-1, 33) for b in dst.bins])
    assert_close(got, Bo, "C1")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]


def test_custom_registry_aliasing(oracle):
    """Non-standard registry: a==dest cross pair, 3-category pair, repeated dest."""
    pairs = [fsbm.InteractionPair("gl", 5, 0, 5), fsbm.InteractionPair("sl", 4, 0, 5),
             fsbm.InteractionPair("ll", 0, 0, 0), fsbm.InteractionPair("il", 1, 0, 0)]
    ctx, grid, tabs = make_ctx(33, pairs=pairs, coeff=0.1)
    st, mask, B = thunder_host(oracle, ctx, 3, 3, 4, 1.0, 9)
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=0.5)
    assert s == 0
    for numerics in ("exact", "fast"):
        st2 = fsbm.GridState(st.ranges, grid, st.temperature, st.pressure, [b.copy() for b in st.bins])
        fsbm.fissioned_step(st2, None, fsbm.StepContext(ctx, fsbm.CoalConfig(0.5)),
                            fsbm.ExecPlan(numerics=numerics))
        got = np.stack([b.reshape(-1, 33) for b in st2.bins])
        if numerics == "exact":
            assert np.array_equal(got, Bo)
        else:
            assert_close(got, Bo, "custom registry")


@pytest.mark.parametrize("numerics", ["exact", "fast"])
def test_stiffness_first_point(oracle, numerics):
    ctx, grid, tabs = make_ctx(33, coeff=1500.0)
    st, mask, B = thunder_host(oracle, ctx, 3, 4, 5, 0.5, 11)
    s, _, err_o, _ = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 4
    with pytest.raises(fsbm.StiffnessError) as ei:
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics=numerics))
    e = ei.value
    assert e.point == tuple(int(v) for v in err_o[2:5])
    assert (e.category, e.bin) == (int(err_o[0]), int(err_o[1]))


def test_stiffness_tile_order(oracle):
    """With patches/tiles the reported point is the first in (tile, j, k, i) order."""
    ctx, grid, tabs = make_ctx(33, coeff=1500.0)
    st, mask, B = thunder_host(oracle, ctx, 4, 2, 4, 1.0, 5)
    tiles = fsbm.decompose(st.ranges, 2, 2)
    x, abd, t750, t500, g = oracle_inputs(oracle, ctx, tabs)
    want = None
    for t, (its, ite, jts, jte) in enumerate(tiles.tiles):  # run_chunks order per tile
        for j in range(jts, jte + 1):
            for k in range(1, st.ranges.nk() + 1):
                for i in range(its, ite + 1):
                    p = st.point_index(i, k, j)
                    if want is None and mask[p]:
                        b = np.ascontiguousarray(B[:, p])
                        s, _, ce = oracle.coal_step(x, abd, t750, t500, g, b, float(st.pressure[p]))
                        if s == 4:
                            want = ((i, k, j), ce)
    assert want is not None
    with pytest.raises(fsbm.StiffnessError) as ei:
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, tiles=tiles), fsbm.ExecPlan())
    assert ei.value.point == want[0]
    assert (ei.value.category, ei.value.bin) == want[1]


def test_errors_and_edge_cases():
    ctx, grid, _ = make_ctx(33)
    T = np.full(4 * 3 * 2, 250.0)
    P = np.full_like(T, 600.0)
    bins = [np.zeros(T.size * 33) for _ in range(6)]
    st = fsbm.GridState(fsbm.Ranges(1, 4, 1, 3, 1, 2), grid, T, P, bins)
    # collapse 3 with automatic scratch -> ConfigError (driver.cpp:213-221)
    with pytest.raises(fsbm.ConfigError):
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx),
                            fsbm.ExecPlan("parallel", 3, 2, "on_demand", "automatic"))
    with pytest.raises(fsbm.ConfigError):
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), fsbm.ExecPlan(threads=0))
    # stale mask -> DomainError (driver.cpp:361-367)
    bad = fsbm.PredicateMask(st.ranges, np.zeros(T.size, np.uint8), 0)
    with pytest.raises(fsbm.DomainError):
        fsbm.fissioned_step(st, bad, fsbm.StepContext(ctx), fsbm.ExecPlan())
    # mask extents mismatch -> ShapeError
    with pytest.raises(fsbm.ShapeError):
        fsbm.fissioned_step(st, fsbm.PredicateMask(fsbm.Ranges(1, 2, 1, 1, 1, 1), None),
                            fsbm.StepContext(ctx), fsbm.ExecPlan())
    # dt <= 0 -> DomainError (coal_step argument check)
    with pytest.raises(fsbm.DomainError):
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, fsbm.CoalConfig(0.0)), fsbm.ExecPlan())
    # all-cold state: nothing runs, dt is never checked, bitwise identity
    st.temperature[:] = 100.0
    st.bins[0][:] = 1.0
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, fsbm.CoalConfig(-1.0), cnt), fsbm.ExecPlan())
    assert (st.bins[0] == 1.0).all() and cnt.points == 0
    # all-zero spectra at warm points: pairs all skipped, identity, zero triples
    st.temperature[:] = 260.0
    st.bins[0][:] = 0.0
    fsbm.fissioned_step(st, None, fsbm.StepContext(ctx, counters=cnt), fsbm.ExecPlan())
    assert all((b == 0).all() for b in st.bins) and cnt.triples == 0 and cnt.points == T.size


def test_fast_is_deterministic_and_host_equals_device(oracle):
    ctx, grid, tabs = make_ctx(33)
    st, mask, B = thunder_host(oracle, ctx, 4, 5, 6, 0.8, 21)
    outs = []
    for _ in range(2):
        d = device_state(st)
        fsbm.fissioned_step(d, None, fsbm.StepContext(ctx), fsbm.ExecPlan())
        outs.append(np.stack([b.cpu().numpy() for b in d.bins]))
    h = fsbm.GridState(st.ranges, grid, st.temperature, st.pressure, [b.copy() for b in st.bins])
    fsbm.fissioned_step(h, None, fsbm.StepContext(ctx), fsbm.ExecPlan())
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], np.stack(h.bins))


def test_device_generator_and_conservation_at_scale(oracle):
    """Size-independent properties at a larger size: per-point mass conservation,
    number non-increase, and sampled points vs the oracle on the same input bytes."""
    import torch
    ctx, grid, tabs = make_ctx(33)
    st, mask = synth.thunderstorm_device(ctx, 40, 20, 50, 1.0, 42)
    nkr = 33
    B0 = torch.stack([b.view(-1, nkr) for b in st.bins]).cpu().numpy()
    # the device generator agrees with the oracle's restatement of the builder
    for p in (0, 123, 39999):
        np.testing.assert_allclose(B0[:, p], oracle.thunderstorm_point(grid.x, 42, p), rtol=1e-14)
    fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx), fsbm.ExecPlan())
    B1 = torch.stack([b.view(-1, nkr) for b in st.bins]).cpu().numpy()
    m0 = (B0 * grid.x).sum(axis=(0, 2))
    m1 = (B1 * grid.x).sum(axis=(0, 2))
    assert np.all(np.abs(m1 - m0) <= 1e-12 * m0)
    assert np.all(B1.sum(axis=(0, 2)) <= B0.sum(axis=(0, 2)) * (1 + 1e-15))
    x, abd, t750, t500, g = oracle_inputs(oracle, ctx, tabs)
    P = st.pressure.cpu().numpy()
    for p in (0, 7, 12345, 39999):
        b = np.ascontiguousarray(B0[:, p])
        assert oracle.coal_step(x, abd, t750, t500, g, b, float(P[p]))[0] == 0
        assert_close(B1[:, p], b, f"point {p}")


@pytest.mark.parametrize("nkr,ratio,pmode", [
    (33, None, "levels"),     # level pressure, groups straddling levels: 1-2 slots per batch
    (33, None, "random"),     # per-point pressure: general (K500 + w*Kd as a K=72 GEMM)
    (33, 1.7, "random"),      # non-doubling grid: exception (non owner-local) cells
    (33, 2.2, "levels"),
    (32, None, "levels"),     # no top-row tile
    (32, 1.9, "random"),
])
def test_fast_pressure_fields_and_grids(oracle, nkr, ratio, pmode):
    """FAST path against the oracle on every point of a multi-batch grid, for uniform,
    mixed and per-point pressure weights and for grids with exception cells."""
    ctx, grid, tabs = make_ctx(nkr, ratio=ratio)
    st, mask, B = thunder_host(oracle, ctx, 5, 7, 37, 0.9, 5)
    if pmode == "random":
        rng = np.random.default_rng(11)
        st.pressure[:] = rng.uniform(350.0, 950.0, st.pressure.shape)
        st.pressure[::7] = 600.0  # some exact repeats
    s, cnt_o, _, Bo = run_oracle_grid(oracle, ctx, tabs, st, mask, B, dt=0.3)
    assert s == 0
    dst = device_state(st)
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(dst, None, fsbm.StepContext(ctx, fsbm.CoalConfig(0.3, 1), cnt), fsbm.ExecPlan())
    got = np.stack([b.cpu().numpy().reshape(-1, nkr) for b in dst.bins])
    assert_close(got, Bo, f"nkr{nkr} ratio{ratio} {pmode}")
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == [int(v) for v in cnt_o]


@pytest.mark.parametrize("kernel,nkr", [("direct", 33), ("dmma", 33), ("dmmag", 33), ("dmmag", 66),
                                        ("direct", 66), ("dmmag", 132)])
def test_stiffness_lowest_bin_every_fast_kernel(oracle, monkeypatch, kernel, nkr):
    """A strongly stiff step (many bins of many categories fail at every point): each FAST
    kernel must report the reference's first point AND its first (category, bin) -- every
    failing bin reaches the sink, whichever warp sees it first (coalescence.cpp:313-328;
    repeated launches, so a scheduling-dependent skip would show)."""
    monkeypatch.setenv("FSBM_FAST_KERNEL", kernel)
    ctx, grid, tabs = make_ctx(nkr, coeff=20000.0)
    st, mask, B = thunder_host(oracle, ctx, 2, 3, 11, 1.0, 23)
    s, _, err_o, _ = run_oracle_grid(oracle, ctx, tabs, st, mask, B)
    assert s == 4
    want = (tuple(int(v) for v in err_o[2:5]), int(err_o[0]), int(err_o[1]))
    for _ in range(5):
        d = device_state(st)
        with pytest.raises(fsbm.StiffnessError) as ei:
            fsbm.fissioned_step(d, None, fsbm.StepContext(ctx), fsbm.ExecPlan())
        e = ei.value
        assert (e.point, e.category, e.bin) == want, kernel
