"""The C restatement (oracle/coal_oracle.c) pinned against the real reference
(oracle/_ref) and the SPEC.md known-answer examples.  CPU only."""
import numpy as np
import pytest

from pyoracle import equal_range_ratio


def test_spec_hand_oracles(oracle, golden):
    # [2,0] -> [1.6,0.2]; [0,1,0] -> [0,0.9,0.05] (tolerance 1e-15)
    for name, x, init, want in (("two_bin", [1.0, 2.0], [2.0, 0.0], [1.6, 0.2]),
                                ("three_bin", [1.0, 2.0, 4.0], [0.0, 1.0, 0.0], [0.0, 0.9, 0.05])):
        x = np.array(x)
        g = oracle.gain_table(x, 2.0)
        n = len(x)
        abd = np.array([0, 0, 0], np.int32)
        t750, t500 = np.ones(n * n), np.ones(n * n)
        b = np.zeros((6, n))
        b[0] = init
        st, cnt, _ = oracle.coal_step(x, abd, t750, t500, g, b, 600.0, dt=0.1)
        assert st == 0
        np.testing.assert_allclose(b[0], want, rtol=0, atol=1e-15)
        assert np.array_equal(b[0], golden[f"hand_{name}_out"])  # bitwise == real reference
        assert np.array_equal(cnt, golden[f"hand_{name}_counters"])


def test_spec_table_and_interp_examples(oracle):
    x = np.array([1.0, 2.0])
    t750, t500 = oracle.build_tables(x, npairs=1, family=1, coeff=1.0, level_scale=1.5)
    assert list(t750) == [2, 3, 3, 4] and list(t500) == [3, 4.5, 4.5, 6]
    w = oracle.pressure_weight(625.0)
    assert oracle.interpolate(t750[3], t500[3], w) == 5.0 and w == 0.5
    assert oracle.interpolate(t750[2], t500[2], w) == 3.75
    assert oracle.pressure_weight(300) == 0.0 and oracle.pressure_weight(900) == 1.0


@pytest.mark.parametrize("nkr", [2, 17, 33, 66, 132, 264])
def test_grid_gain_tables_bitwise(oracle, reference, nkr):
    r = equal_range_ratio(nkr) if nkr > 2 else 2.0
    xo = oracle.mass_grid(nkr, 3.35e-14, r)
    assert np.array_equal(xo, reference.mass_grid(nkr, 3.35e-14, r))
    go = oracle.gain_table(xo, r)
    gr = reference.gain_table(nkr, 3.35e-14, r)
    for a, b in zip(go, gr):
        assert np.array_equal(a, b)


def test_golden_gain_tables(oracle, golden):
    for nkr in (17, 33, 66):
        r = equal_range_ratio(nkr)
        go = oracle.gain_table(oracle.mass_grid(nkr, 3.35e-14, r), r)
        for a, key in zip(go, ("lo", "wlo", "whi", "top")):
            assert np.array_equal(a, golden[f"gain_nkr{nkr}_{key}"])


@pytest.mark.parametrize("family", [0, 1, 2, 3])
def test_build_tables_bitwise(oracle, reference, family):
    nkr = 33
    x = oracle.mass_grid(nkr)
    a = oracle.build_tables(x, family=family, coeff=0.7, pair_scale_step=0.05)
    b = reference.build_tables(nkr, family=family, coeff=0.7, pair_scale_step=0.05)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_golden_points_bitwise(oracle, golden):
    for nkr in (17, 33, 66):
        r = equal_range_ratio(nkr)
        x = oracle.mass_grid(nkr, 3.35e-14, r)
        g = oracle.gain_table(x, r)
        abd = oracle.default_registry()
        t750, t500 = oracle.build_tables(x, pair_scale_step=0.05)
        pin = golden[f"point_nkr{nkr}_in"]
        for q, pres in enumerate(golden[f"point_nkr{nkr}_pressure"]):
            b = pin[q].copy()
            st, cnt, _ = oracle.coal_step(x, abd, t750, t500, g, b, pres, dt=1.0,
                                          substeps=2 if q == 1 else 1)
            assert st == 0
            assert np.array_equal(b, golden[f"point_nkr{nkr}_out"][q])
            assert np.array_equal(cnt, golden[f"point_nkr{nkr}_counters"][q])


@pytest.mark.parametrize("kstrat", [0, 1])
@pytest.mark.parametrize("substeps", [1, 3])
def test_coal_step_vs_reference(oracle, reference, kstrat, substeps):
    nkr = 33
    x = oracle.mass_grid(nkr)
    g = oracle.gain_table(x, 2.0)
    abd = oracle.default_registry()
    t750, t500 = oracle.build_tables(x, pair_scale_step=0.05)
    for p in (0, 5, 99):
        b = oracle.thunderstorm_point(x, 7, p)
        b[3] = 0.0  # one empty category exercises the all_zero pair skip
        b2 = b.copy()
        s1 = oracle.coal_step(x, abd, t750, t500, g, b, 540.0 + 20 * p % 300, dt=0.7,
                              substeps=substeps, kernel_strategy=kstrat)
        s2 = reference.coal_step(nkr, t750, t500, b2, 540.0 + 20 * p % 300, dt=0.7,
                                 substeps=substeps, kernel_strategy=kstrat)
        assert s1[0] == s2[0] == 0
        assert np.array_equal(s1[1], s2[1])
        assert np.array_equal(b, b2)


def test_stiffness_matches_reference(oracle, reference):
    nkr = 33
    x = oracle.mass_grid(nkr)
    g = oracle.gain_table(x, 2.0)
    abd = oracle.default_registry()
    t750, t500 = oracle.build_tables(x, coeff=1500.0)
    b = oracle.thunderstorm_point(x, 42, 3)
    b2 = b.copy()
    s1 = oracle.coal_step(x, abd, t750, t500, g, b, 800.0, dt=1.0)
    s2 = reference.coal_step(nkr, t750, t500, b2, 800.0, dt=1.0)
    assert s1[0] == s2[0] == 4
    assert s1[2] == s2[2]
    assert np.array_equal(b, b2)  # identical partial mutation


def test_synthetic_case_and_mask(oracle, reference, golden):
    T1, P1, B1 = oracle.synthetic_case(6, 5, 7, 0.3, 42, 33)
    T2, P2, B2 = reference.synthetic_case(6, 5, 7, 0.3, 42, 33)
    assert np.array_equal(T1, T2) and np.array_equal(P1, P2) and np.array_equal(B1, B2)
    T, _, _ = oracle.synthetic_case(10, 10, 10, 0.3, 42, 33)
    mask, n = oracle.fission_predicates(T)
    assert n == 300 == int(golden["mask_10cube_count"])
    assert np.array_equal(mask, golden["mask_10cube"])


@pytest.mark.parametrize("threads", [1, 3])
def test_step_grid_vs_fissioned_step(oracle, reference, golden, threads):
    ni, nk, nj, nkr = 4, 5, 6, 33
    T, P, B = golden["grid_T"], golden["grid_P"], golden["grid_in"].copy()
    x = oracle.mass_grid(nkr)
    g = oracle.gain_table(x, 2.0)
    abd = oracle.default_registry()
    t750, t500 = oracle.build_tables(x, pair_scale_step=0.05)
    mask, _ = oracle.fission_predicates(T)
    st, cnt, err = oracle.step_grid(ni, nk, nj, x, abd, t750, t500, g, mask, P, B,
                                    nthreads=threads)
    assert st == 0
    assert np.array_equal(B, golden["grid_out"])
    assert np.array_equal(cnt, golden["grid_counters"])


def test_mass_conservation_oracle(oracle):
    nkr = 33
    x = oracle.mass_grid(nkr)
    g = oracle.gain_table(x, 2.0)
    abd = oracle.default_registry()
    t750, t500 = oracle.build_tables(x, pair_scale_step=0.05)
    b = oracle.thunderstorm_point(x, 1, 11)
    m0 = float((b * x).sum())
    n0 = float(b.sum())
    for _ in range(4):  # the thunderstorm input turns stiff (snow) at step 5 with dt=1
        assert oracle.coal_step(x, abd, t750, t500, g, b, 700.0)[0] == 0
    assert abs(float((b * x).sum()) - m0) <= 1e-12 * m0
    assert float(b.sum()) <= n0
