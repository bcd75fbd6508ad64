"""Known-answer tests pinning the Bott (1998) flux-method oracle (oracle/bott_oracle.c).

The reference does not implement Bott's scheme, so there is no reference
output to compare with; these tests pin the restatement instead:
  * SPEC.md:206-207 hand examples (products landing in the top bin behave exactly like
    the reference's top rule),
  * an independent pure-Python restatement of the same loop (bitwise: same libm calls,
    same operation order, no FMA in either),
  * Bott's eq. 13 in its literal two-exponential form (the oracle uses the
    cancellation-free expm1 form),
  * positivity under very stiff steps, mass conservation to round-off, counters,
  * the Golovin kernel's analytic number decay N(t) = N0 exp(-b M t).
CPU only."""
import math

import numpy as np
import pytest

from pyoracle import equal_range_ratio


def _tables(oracle, x, family=1, coeff=1.0, level_scale=1.5, pair_scale_step=0.05, npairs=20):
    return oracle.build_tables(x, npairs=npairs, family=family, coeff=coeff, level_scale=level_scale,
                               pair_scale_step=pair_scale_step)


def py_bott_step(x, abd, t750, t500, lo, cour, bins6, pressure, dt, substeps):
    """Independent pure-Python restatement of orc_bott_step (small cases only)."""
    nkr = len(x)
    w = min(max((pressure - 500.0) / (750.0 - 500.0), 0.0), 1.0)
    g = [[bins6[c][k] * x[k] for k in range(nkr)] for c in range(6)]
    rx = [1.0 / v for v in x]
    dts = dt / substeps
    for _ in range(substeps):
        for p in range(len(abd) // 3):
            a, b, d = abd[3 * p], abd[3 * p + 1], abd[3 * p + 2]
            if all(v == 0.0 for v in g[a]):
                continue
            self_ = a == b
            for i in range(nkr):
                for j in range(i if self_ else 0, nkr):
                    gai, gbj = g[a][i], g[b][j]
                    if gai == 0.0 or gbj == 0.0:
                        continue
                    e = (p * nkr + i) * nkr + j
                    ck = (t500[e] + (t750[e] - t500[e]) * w) * dts
                    diag = self_ and i == j
                    if diag:
                        ck *= 0.5
                    z = min(ck * gai * gbj, gai * x[j], gbj * x[i])
                    if diag:
                        gsk = min(2.0 * (z * rx[i]), gai)
                        g[a][i] = gai - gsk
                    else:
                        gsi, gsj = min(z * rx[j], gai), min(z * rx[i], gbj)
                        g[a][i] = gai - gsi
                        g[b][j] = g[b][j] - gsj
                        gsk = gsi + gsj
                    k = int(lo[i * nkr + j])
                    if k < 0:
                        g[d][nkr - 1] += gsk
                        continue
                    gk, gkp = g[d][k] + gsk, g[d][k + 1]
                    if gk > 0.0:
                        c = cour[i * nkr + j]
                        q = 1.0 / gk
                        u, r, lg = (gkp - gk) * q, gkp * q, -138.15510557964274
                        x1 = math.log1p(u) if -0.5 < u < 0.5 else math.log(r + 1e-60)
                        x1 = min(max(x1, lg), -lg)
                        fl = gsk * c if x1 == 0.0 else gsk * math.exp(x1 * (0.5 - c)) * math.expm1(x1 * c) / x1
                        fl = min(fl, gsk)
                        g[d][k] = gk - fl
                        g[d][k + 1] = gkp + fl
                    else:
                        g[d][k] = gk
    return np.array([[g[c][k] * rx[k] for k in range(nkr)] for c in range(6)])


def test_bott_spec_top_bin_examples(oracle):
    """The SPEC.md:206-207 inputs (K = 1, dt = 0.1), derived by hand for Bott's Gauss-Seidel
    sweep; every product lands in the top bin (mass-conserving top rule).
    [2,0]: (0,0) z = 0.05*2*2, gsk = 0.4 -> g = [1.6, 0.4]; (0,1) now sees bin 1 (Gauss-Seidel;
           Kovetz-Olund's Jacobi sweep does not, hence its [1.6, 0.2]): z = 0.1*1.6*0.4 = 0.064,
           gsi = 0.032, gsj = 0.064 -> top: g = [1.568, 0.432] -> n = [1.568, 0.216].
    [0,1,0]: (1,1) z = 0.2, gsk = 0.2 -> g = [0, 1.8, 0.2]; (1,2) z = 0.1*1.8*0.2 = 0.036,
           gsi = 0.009, gsj = 0.018 -> g = [0, 1.791, 0.209] -> n = [0, 0.8955, 0.05225]."""
    for x, init, want in (([1.0, 2.0], [2.0, 0.0], [1.568, 0.216]),
                          ([1.0, 2.0, 4.0], [0.0, 1.0, 0.0], [0.0, 0.8955, 0.05225])):
        x = np.array(x)
        lo = oracle.gain_table(x, 2.0)[0]
        cour = oracle.bott_courant(x, lo)
        n = len(x)
        b = np.zeros((6, n))
        b[0] = init
        st, cnt = oracle.bott_step(x, np.array([0, 0, 0], np.int32), np.ones(n * n), np.ones(n * n), lo,
                                   cour, b, 600.0, dt=0.1)
        assert st == 0
        np.testing.assert_allclose(b[0], want, rtol=0, atol=1e-15)
        assert (b[0] * x).sum() == pytest.approx((np.array(init) * x).sum(), rel=1e-15)
        assert list(cnt) == [n * (n + 1) // 2, 1, n * (n + 1) // 2]


def test_bott_hand_flux_case(oracle):
    """One cross pair liquid + ice1 -> ice1 on x = [1,2,4,8] (K = 1, dt = 0.1), liquid n = [1,0,0,0],
    ice1 n = [0,1,1,0]; the sweep written out by hand with Bott's literal eq. 13:
      (0,1): z = 0.1*1*2 = 0.2 -> gsi = 0.1 (liquid 0), gsj = 0.2 (ice1 1), gsk = 0.3 lands at
             m = 3, Courant log2(1.5) in bin 1 -> flux into bin 2 from the exponential profile
             through g1 = 2.1 and g2 = 4.
      (0,2): m = 5 in bin 2 (Courant log2 1.25 < 1/2) with bin 3 empty -> a vanishing flux.
      (0,3): bin 3 now holds that flux: m = 9 >= x3 -> top rule."""
    x = [1.0, 2.0, 4.0, 8.0]
    xa = np.array(x)
    lo = oracle.gain_table(xa, 2.0)[0]
    cour = oracle.bott_courant(xa, lo)
    assert cour[1] == pytest.approx(math.log2(1.5), abs=1e-15)
    b = np.zeros((6, 4))
    b[0] = [1.0, 0.0, 0.0, 0.0]
    b[1] = [0.0, 1.0, 1.0, 0.0]
    oracle.bott_step(xa, np.array([0, 1, 1], np.int32), np.ones(16), np.ones(16), lo, cour, b, 600.0, dt=0.1)

    def eq13(gsk, gk, gkp, c):
        x1 = math.log(gkp / gk + 1e-60)
        return min(gsk / x1 * (math.exp(0.5 * x1) - math.exp(x1 * (0.5 - c))), gsk)

    ga = [1.0, 0.0, 0.0, 0.0]
    gd = [0.0, 2.0, 4.0, 0.0]  # ice1 as mass: n * x
    for j, k in ((1, 1), (2, 2), (3, -1)):
        z = min(0.1 * ga[0] * gd[j], ga[0] * x[j], gd[j] * x[0])
        gsi, gsj = z / x[j], z / x[0]
        ga[0] -= gsi
        gd[j] -= gsj
        gsk = gsi + gsj
        if k < 0:
            gd[3] += gsk
            continue
        gk = gd[k] + gsk
        fl = eq13(gsk, gk, gd[k + 1], math.log((x[0] + x[j]) / x[k]) / math.log(2.0))
        gd[k], gd[k + 1] = gk - fl, gd[k + 1] + fl
    assert 0.0 < gd[3] < 1e-12  # (0,2) moved a vanishing flux, (0,3) then collided with it
    np.testing.assert_allclose(b[0], np.array(ga) / xa, rtol=1e-13, atol=0)
    np.testing.assert_allclose(b[1], np.array(gd) / xa, rtol=1e-12, atol=0)


def test_bott_flux_is_eq13(oracle):
    # the cancellation-free form equals Bott's literal eq. 13 gsk/x1 (e^{x1/2} - e^{x1(1/2-c)})
    rng = np.random.default_rng(5)
    for _ in range(200):
        gk, gkp = rng.uniform(0.1, 10.0, 2)
        c, gsk = rng.uniform(0.0, 1.0), rng.uniform(0.0, gk)
        x1 = math.log(gkp / gk)
        lit = min(gsk / x1 * (math.exp(0.5 * x1) - math.exp(x1 * (0.5 - c))), gsk)
        assert oracle.bott_flux(gsk, gk, gkp, c) == pytest.approx(lit, rel=1e-12, abs=1e-300)
    # limits: equal neighbours -> flux = gsk c; empty upper bin -> x1 = ln(1e-60)
    assert oracle.bott_flux(0.5, 2.0, 2.0, 0.25) == 0.125
    assert 0.0 <= oracle.bott_flux(0.5, 2.0, 0.0, 0.3) <= 0.5


@pytest.mark.parametrize("nkr,substeps", [(8, 1), (12, 2)])
def test_bott_oracle_matches_python_restatement(oracle, nkr, substeps):
    x = oracle.mass_grid(nkr, 3.35e-14, equal_range_ratio(nkr) if nkr > 2 else 2.0)
    ratio = equal_range_ratio(nkr)
    lo = oracle.gain_table(x, ratio)[0]
    cour = oracle.bott_courant(x, lo)
    abd = oracle.default_registry()
    t750, t500 = _tables(oracle, x, coeff=3.0e3)
    rng = np.random.default_rng(nkr)
    for trial in range(3):
        b = rng.uniform(0.0, 1e3, (6, nkr))
        b[rng.uniform(size=(6, nkr)) < 0.3] = 0.0
        P = float(rng.uniform(400.0, 900.0))
        want = py_bott_step(x, list(abd), t750, t500, lo, cour, b.copy(), P, 1.0, substeps)
        st, _ = oracle.bott_step(x, abd, t750, t500, lo, cour, b, P, dt=1.0, substeps=substeps)
        assert st == 0
        assert np.array_equal(b, want), np.abs(b - want).max()


def _thunder(oracle, nkr, n, seed=42):
    x = oracle.mass_grid(nkr, 3.35e-14, equal_range_ratio(nkr))
    b = oracle.thunderstorm_block(x, seed, 0, n).reshape(6, n, nkr)
    return x, np.ascontiguousarray(b)


def test_bott_positive_and_mass_conserving(oracle):
    nkr, n = 33, 24
    x, b = _thunder(oracle, nkr, n)
    lo = oracle.gain_table(x, 2.0)[0]
    cour = oracle.bott_courant(x, lo)
    abd = oracle.default_registry()
    P = np.linspace(400.0, 900.0, n)
    for coeff, steps in ((1.0, 20), (1500.0, 3), (1e7, 2)):  # mild, stiff for Kovetz-Olund, extreme
        t750, t500 = _tables(oracle, x, coeff=coeff)
        bb = b.copy()
        m0 = (bb * x).sum(axis=2)
        for _ in range(steps):
            st, cnt = oracle.bott_step_grid(x, abd, t750, t500, lo, cour, None, P, bb, dt=1.0)
            assert st == 0
        assert (bb >= 0.0).all()  # positive-definite (no StiffnessError possible)
        m1 = (bb * x).sum(axis=2)
        np.testing.assert_allclose(m1.sum(0), m0.sum(0), rtol=1e-13)  # per point, all categories
        assert (bb.sum(axis=(0, 2)) <= b.sum(axis=(0, 2)) * (1 + 1e-12)).all() or coeff > 1.0


def test_bott_counters_match_coal_step(oracle):
    nkr = 33
    x, b = _thunder(oracle, nkr, 4)
    g = oracle.gain_table(x, 2.0)
    cour = oracle.bott_courant(x, g[0])
    abd = oracle.default_registry()
    t750, t500 = _tables(oracle, x)
    for ks in (0, 1):
        for sub in (1, 3):
            b1, b2 = b[:, 0].copy(), b[:, 0].copy()
            _, c_ko, _ = oracle.coal_step(x, abd, t750, t500, g, b1, 700.0, substeps=sub, kernel_strategy=ks)
            _, c_bo = oracle.bott_step(x, abd, t750, t500, g[0], cour, b2, 700.0, substeps=sub,
                                       kernel_strategy=ks)
            assert list(c_ko) == list(c_bo)


def test_bott_golovin_number_decay(oracle):
    """Golovin kernel K = b (x_i + x_j): the continuous SCE has N(t) = N0 exp(-b M t)
    exactly.  On a fine mass grid Bott's scheme follows it (Bott 1998, Fig. 2)."""
    nkr = 132
    ratio = equal_range_ratio(nkr)
    x = oracle.mass_grid(nkr, 3.35e-14, ratio)
    lo = oracle.gain_table(x, ratio)[0]
    cour = oracle.bott_courant(x, lo)
    bcoef = 1500.0
    t750, t500 = oracle.build_tables(x, npairs=1, family=1, coeff=bcoef, level_scale=1.0,
                                     pair_scale_step=0.0)
    abd = np.array([0, 0, 0], np.int32)
    b = np.zeros((6, nkr))
    b[0] = oracle.exponential_init(x, 1e8, x[30])
    N0, M = b[0].sum(), (b[0] * x).sum()
    t, dt = 0.0, 0.02
    Kscale = np.mean(t750.reshape(nkr, nkr)[0, :2] / (x[0] + x[:2]))  # = b of family 1
    for _ in range(40):
        oracle.bott_step(x, abd, t750, t500, lo, cour, b, 600.0, dt=dt)
        t += dt
    want = N0 * math.exp(-Kscale * M * t)
    assert 0.2 < want / N0 < 0.8  # a real test: the population changed substantially
    assert b[0].sum() == pytest.approx(want, rel=0.05)
    assert (b[0] * x).sum() == pytest.approx(M, rel=1e-12)
