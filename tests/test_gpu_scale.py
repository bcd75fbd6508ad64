"""GPU parity at scale and over many steps (SPEC.md acceptance criteria 1, 2, 4), through
the C ABI, against the unmodified reference (oracle/_ref) where the reference is the
checker.

Bars: EXACT numerics bitwise equal to the reference; FAST numerics per bin
|gpu - ref| <= 1e-12|ref| + 1e-15 sum_k ref_c[k]; counters exact; per-point mass 1e-12.
"""
import os

import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm
from paper_2409_07232_b200 import synth

pytestmark = pytest.mark.gpu

RTOL, ATOL_FRAC = 1e-12, 1e-15
THREADS = os.cpu_count() or 1


def bar(got, ref):
    """(bins out of tolerance, max |err| / tol)."""
    tol = RTOL * np.abs(ref) + ATOL_FRAC * np.abs(ref).sum(axis=-1, keepdims=True)
    d = np.abs(got - ref)
    return int((d > tol).sum()), float((d / np.maximum(tol, 1e-300)).max())


def ctx_for(nkr, pair_scale_step=0.05, x1=3.35e-14, ratio=None):
    r = ratio or fsbm.equal_range_ratio(nkr)
    grid = fsbm.make_mass_grid(nkr, x1, r)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1.0, 1.5, pair_scale_step))
    return fsbm.CoalContext(grid, tabs), grid, tabs


def to_dev(st):
    import torch
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda:0")
    return fsbm.GridState(st.ranges, st.grid, t(st.temperature), t(st.pressure),
                          [t(b) for b in st.bins])


def bins_np(st, nkr):
    return np.stack([(b.cpu().numpy() if hasattr(b, "cpu") else b).reshape(-1, nkr)
                     for b in st.bins])


def ref_step(reference, dims, nkr, tabs, T, P, B, ratio, dt=1.0, substeps=1, kstrat=1):
    ni, nk, nj = dims
    st, cnt, tim, err = reference.fissioned_step(ni, nk, nj, nkr, tabs.t750.reshape(-1).copy(),
                                                 tabs.t500.reshape(-1).copy(), T, P, B, dt,
                                                 substeps, mode=1, collapse=3, threads=THREADS,
                                                 kernel_strategy=kstrat, scratch_strategy=1,
                                                 ratio=ratio)
    assert st == 0, reference.last_error()
    return [int(v) for v in cnt]


# ---------------------------------------------------------------------------------------
def test_headline_input_200k_points_vs_reference(reference):
    """C2's input builder and tables on a 40 x 50 x 100 grid (200 000 points, all 20
    pairs active): FAST within the bar, EXACT bitwise, counters exact, vs the reference's
    own fissioned_step on the same bytes."""
    import torch
    nkr, dims = 33, (40, 50, 100)
    ctx, grid, tabs = ctx_for(nkr)
    st, mask = synth.thunderstorm_device(ctx, *dims, 1.0, 42)
    B0 = bins_np(st, nkr)
    T, P = st.temperature.cpu().numpy(), st.pressure.cpu().numpy()
    ref = B0.copy()
    cnt_ref = ref_step(reference, dims, nkr, tabs, T, P, ref, grid.ratio)
    assert cnt_ref[1] == 200_000
    for numerics in ("fast", "exact"):
        d = fsbm.GridState(st.ranges, grid, st.temperature, st.pressure,
                           [torch.from_numpy(B0[c].reshape(-1)).cuda() for c in range(6)])
        cnt = fsbm.WorkCounters()
        fsbm.fissioned_step(d, mask, fsbm.StepContext(ctx, counters=cnt),
                            fsbm.ExecPlan("parallel", 3, 8, "on_demand", "arena", numerics))
        got = bins_np(d, nkr)
        assert [cnt.triples, cnt.points, cnt.kernel_evals] == cnt_ref
        if numerics == "exact":
            assert np.array_equal(got, ref)
        else:
            bad, worst = bar(got, ref)
            assert bad == 0, (bad, worst)
            m0, m1 = (B0 * grid.x).sum(axis=(0, 2)), (got * grid.x).sum(axis=(0, 2))
            assert np.all(np.abs(m1 - m0) <= 1e-12 * m0)


@pytest.mark.parametrize("nkr,dims", [(66, (2, 40, 100)), (132, (2, 40, 80)), (264, (1, 40, 125))])
def test_wide_bins_5k_points_vs_reference(reference, nkr, dims):
    """C3/C4/C5 bin counts on >= 5 000 points each (coal_dmmag), FAST and EXACT."""
    import torch
    ctx, grid, tabs = ctx_for(nkr)
    st, mask = synth.thunderstorm_device(ctx, *dims, 1.0, 42)
    B0 = bins_np(st, nkr)
    T, P = st.temperature.cpu().numpy(), st.pressure.cpu().numpy()
    ref = B0.copy()
    cnt_ref = ref_step(reference, dims, nkr, tabs, T, P, ref, grid.ratio)
    assert cnt_ref[1] >= 5000
    for numerics in ("fast", "exact"):
        d = fsbm.GridState(st.ranges, grid, st.temperature, st.pressure,
                           [torch.from_numpy(B0[c].reshape(-1)).cuda() for c in range(6)])
        cnt = fsbm.WorkCounters()
        fsbm.fissioned_step(d, mask, fsbm.StepContext(ctx, counters=cnt),
                            fsbm.ExecPlan(numerics=numerics))
        got = bins_np(d, nkr)
        assert [cnt.triples, cnt.points, cnt.kernel_evals] == cnt_ref
        if numerics == "exact":
            assert np.array_equal(got, ref)
        else:
            bad, worst = bar(got, ref)
            assert bad == 0, (bad, worst)


# ---- SPEC acceptance criterion 1: 20-step variant equivalence ---------------------------
@pytest.mark.parametrize("dims", [(16, 8, 8), (32, 16, 10)])
@pytest.mark.parametrize("nkr", [17, 33])
def test_spec1_twenty_steps_vs_reference(reference, dims, nkr):
    """make_synthetic_case (liquid-only, reference default tables), cloud fractions
    {0, 0.3, 1} x seeds {1, 42}, 20 steps: EXACT bitwise equal to the reference's
    fissioned_step after every step; FAST within the bar after 20 steps."""
    grid = fsbm.make_mass_grid(nkr)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry())  # reference defaults
    ctx = fsbm.CoalContext(grid, tabs)
    for cf in (0.0, 0.3, 1.0):
        for seed in (1, 42):
            T, P, B = reference.synthetic_case(*dims, cf, seed, nkr)
            ref = B.copy()
            st = fsbm.GridState(fsbm.Ranges(1, dims[0], 1, dims[1], 1, dims[2]), grid, T, P,
                                [B[c].reshape(-1).copy() for c in range(6)])
            ex, fa = to_dev(st), to_dev(st)
            mask = fsbm.fission_predicates(ex, ctx)
            ce, cr = fsbm.WorkCounters(), [0, 0, 0]
            for step in range(20):
                c = ref_step(reference, dims, nkr, tabs, T, P, ref, 2.0)
                cr = [a + b for a, b in zip(cr, c)]
                fsbm.fissioned_step(ex, mask, fsbm.StepContext(ctx, counters=ce),
                                    fsbm.ExecPlan("parallel", 3, 4, "on_demand", "arena", "exact"))
                fsbm.fissioned_step(fa, mask, fsbm.StepContext(ctx),
                                    fsbm.ExecPlan("parallel", 3, 4, "on_demand", "arena", "fast"))
                assert np.array_equal(bins_np(ex, nkr), ref), (cf, seed, step)
            assert [ce.triples, ce.points, ce.kernel_evals] == cr
            bad, worst = bar(bins_np(fa, nkr), ref)
            assert bad == 0, (cf, seed, bad, worst)


# ---- SPEC acceptance criterion 2: 100-step Golovin mass conservation -------------------
@pytest.mark.parametrize("numerics", ["fast", "exact"])
def test_spec2_hundred_steps_mass_and_number(reference, numerics):
    import math
    nkr, dims = 33, (8, 8, 8)
    grid = fsbm.make_mass_grid(nkr)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry())
    ctx = fsbm.CoalContext(grid, tabs)
    T, P, B = reference.synthetic_case(*dims, 1.0, 42, nkr)
    st = to_dev(fsbm.GridState(fsbm.Ranges(1, 8, 1, 8, 1, 8), grid, T, P,
                               [B[c].reshape(-1).copy() for c in range(6)]))
    mask = fsbm.fission_predicates(st, ctx)

    def totals():
        b = bins_np(st, nkr)
        return math.fsum((b * grid.x).reshape(-1)), math.fsum(b.reshape(-1))

    m0, n_prev = totals()
    for _ in range(100):
        fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics=numerics))
        m, n = totals()
        assert n < n_prev  # strictly non-increasing
        n_prev = n
    assert abs(m - m0) <= 1e-12 * m0


# ---- SPEC acceptance criterion 4: first-order substep convergence ------------------------
def test_spec4_substep_convergence():
    import torch
    nkr = 33
    grid = fsbm.make_mass_grid(nkr)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry())
    ctx = fsbm.CoalContext(grid, tabs)
    st0 = synth.liquid_case_host(4, 4, 4, 1.0, 42, grid)

    def run(s):
        d = to_dev(st0)
        fsbm.fissioned_step(d, None, fsbm.StepContext(ctx, fsbm.CoalConfig(1.0, s)),
                            fsbm.ExecPlan())
        return bins_np(d, nkr)

    fine = run(16 * 8)
    err = [np.abs(run(s) - fine).sum() for s in (1, 2, 4, 8)]
    ratios = [err[q] / err[q + 1] for q in range(3)]
    assert all(1.7 <= r <= 2.3 for r in ratios), ratios


# ---- paths the headline bench does not take ---------------------------------------------
@pytest.mark.parametrize("nkr", [33, 66])
def test_direct_fast_kernel_on_thunderstorm_grid(reference, nkr, monkeypatch):
    """coal_fast (FSBM_FAST_KERNEL=direct) on a thunderstorm grid vs the reference."""
    import torch
    monkeypatch.setenv("FSBM_FAST_KERNEL", "direct")
    ctx, grid, tabs = ctx_for(nkr)
    assert ctx.fast_kernel() == "coal_fast"
    dims = (3, 10, 40)
    st, mask = synth.thunderstorm_device(ctx, *dims, 0.8, 7)
    B0 = bins_np(st, nkr)
    ref = B0.copy()
    cnt_ref = ref_step(reference, dims, nkr, tabs, st.temperature.cpu().numpy(),
                       st.pressure.cpu().numpy(), ref, grid.ratio)
    cnt = fsbm.WorkCounters()
    fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx, counters=cnt), fsbm.ExecPlan())
    bad, worst = bar(bins_np(st, nkr), ref)
    assert bad == 0, (bad, worst)
    assert [cnt.triples, cnt.points, cnt.kernel_evals] == cnt_ref


def test_device_stale_mask_raises():
    """The device path's stale-mask check (flags_kernel, driver.cpp:361-367): a mask that
    disagrees with the temperatures raises DomainError and leaves the state untouched."""
    import torch
    ctx, grid, _ = ctx_for(33)
    st, mask = synth.thunderstorm_device(ctx, 3, 4, 5, 0.5, 3)
    before = bins_np(st, 33)
    bad = fsbm.PredicateMask(st.ranges, mask.call_coal.clone())
    bad.call_coal[7] ^= 1
    with pytest.raises(fsbm.DomainError, match="stale"):
        fsbm.fissioned_step(st, bad, fsbm.StepContext(ctx), fsbm.ExecPlan())
    assert np.array_equal(bins_np(st, 33), before)
    fsbm.fissioned_step(st, mask, fsbm.StepContext(ctx), fsbm.ExecPlan())  # fresh mask: fine


def test_stiffness_message_carries_the_value(reference):
    """StiffnessError text as coalescence.cpp:319-325 ('would become negative (V)') plus
    at_point's coordinates, identical to the reference's message in EXACT numerics."""
    nkr = 33
    grid = fsbm.make_mass_grid(nkr)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1500.0, 1.5, 0.0))
    ctx = fsbm.CoalContext(grid, tabs)
    st0, _ = synth.thunderstorm_device(ctx, 3, 4, 5, 0.5, 11)
    B = bins_np(st0, nkr)
    T, P = st0.temperature.cpu().numpy(), st0.pressure.cpu().numpy()
    ref = B.copy()
    st_ref, _, _, err_ref = reference.fissioned_step(3, 4, 5, nkr, tabs.t750.reshape(-1).copy(),
                                                     tabs.t500.reshape(-1).copy(), T, P, ref,
                                                     1.0, 1, mode=0, collapse=2, threads=1,
                                                     kernel_strategy=1, scratch_strategy=0)
    assert st_ref == 4
    ref_msg = reference.last_error()
    for numerics in ("exact", "fast"):
        st = fsbm.GridState(fsbm.Ranges(1, 3, 1, 4, 1, 5), grid, T.copy(), P.copy(),
                            [B[c].reshape(-1).copy() for c in range(6)])
        with pytest.raises(fsbm.StiffnessError) as ei:
            fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics=numerics))
        e = ei.value
        assert e.point == tuple(int(v) for v in err_ref[2:5])
        assert (e.category, e.bin) == (int(err_ref[0]), int(err_ref[1]))
        assert "would become negative (" in str(e) and e.value < 0
        if numerics == "exact":
            assert str(e) == ref_msg
