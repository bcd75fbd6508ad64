"""CBSNAP01 snapshots (snapshot.cpp) and the GPU digit-agreement comparator (verify.cpp)
against the unmodified reference (oracle/_ref)."""
import os

import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm


def small_state(seed=3, ni=3, nk=4, nj=5, nkr=17):
    rng = np.random.default_rng(seed)
    grid = fsbm.make_mass_grid(nkr, 3.35e-14, fsbm.equal_range_ratio(nkr))
    r = fsbm.Ranges(2, 1 + ni, 1, nk, 3, 2 + nj)
    np_ = r.npoints()
    T = rng.uniform(180, 300, np_)
    P = rng.uniform(400, 900, np_)
    bins = [rng.exponential(1e6, np_ * nkr) * (rng.random(np_ * nkr) < 0.7) for _ in range(6)]
    return fsbm.GridState(r, grid, T, P, bins)


def ranges6(r):
    return [r.ids, r.ide, r.kds, r.kde, r.jds, r.jde]


def test_snapshot_roundtrip_bit_exact(tmp_path):
    s = small_state()
    p = tmp_path / "a.cbsnap"
    fsbm.write_snapshot(s, p)
    t = fsbm.read_snapshot(p)
    assert t.ranges == s.ranges and t.grid.ratio == s.grid.ratio
    assert np.array_equal(t.grid.x, s.grid.x)
    assert np.array_equal(t.temperature, s.temperature) and np.array_equal(t.pressure, s.pressure)
    assert all(np.array_equal(a, b) for a, b in zip(t.bins, s.bins))
    fsbm.write_snapshot(t, tmp_path / "b.cbsnap")
    assert (tmp_path / "a.cbsnap").read_bytes() == (tmp_path / "b.cbsnap").read_bytes()


def test_snapshot_bytes_equal_reference(tmp_path, reference):
    s = small_state(seed=7)
    ours, theirs = tmp_path / "ours.cbsnap", tmp_path / "ref.cbsnap"
    fsbm.write_snapshot(s, ours)
    assert reference.write_snapshot(theirs, ranges6(s.ranges), s.grid.x, s.grid.ratio,
                                    s.temperature, s.pressure, np.stack(s.bins)) == 0
    assert ours.read_bytes() == theirs.read_bytes()
    st, rg, x, ratio, T, P, bins = reference.read_snapshot(ours)
    assert st == 0 and list(rg) == ranges6(s.ranges) and ratio == s.grid.ratio
    assert np.array_equal(bins, np.stack(s.bins)) and np.array_equal(T, s.temperature)


@pytest.mark.parametrize("corrupt,msg", [
    (lambda b: b"XBSNAP01" + b[8:], "is not a coalbench snapshot"),
    (lambda b: b[:8] + (2).to_bytes(4, "little") + b[12:], "unsupported version"),
    (lambda b: b[:12] + (1).to_bytes(4, "little") + b[16:], "implausible nkr"),
    (lambda b: b[:16] + (9).to_bytes(4, "little", signed=True) + b[20:], "invalid domain ranges"),
    (lambda b: b[:-5], "truncated while reading bins"),
    (lambda b: b[:30], "truncated while reading"),
    (lambda b: b + b"\0", "trailing bytes"),
])
def test_snapshot_errors_match_reference(tmp_path, reference, corrupt, msg):
    s = small_state()
    good = tmp_path / "g.cbsnap"
    fsbm.write_snapshot(s, good)
    bad = tmp_path / "bad.cbsnap"
    bad.write_bytes(corrupt(good.read_bytes()))
    with pytest.raises(fsbm.ConfigError, match=msg) as ei:
        fsbm.read_snapshot(bad)
    st = reference.read_snapshot(bad)[0]
    assert st == 3 and reference.last_error() == str(ei.value)


def test_snapshot_missing_file():
    with pytest.raises(fsbm.ConfigError, match="cannot open"):
        fsbm.read_snapshot("/nonexistent/dir/x.cbsnap")


def test_compare_states_shape_errors():
    a, b = small_state(), small_state(ni=4)
    with pytest.raises(fsbm.ShapeError, match="domain ranges differ"):
        fsbm.compare_states(a, b)
    c = small_state(nkr=9)
    with pytest.raises(fsbm.ShapeError, match="nkr differs"):
        fsbm.compare_states(a, c)


def _perturbed(s, rng, rel):
    bins = []
    for b in s.bins:
        b = b.copy()
        b *= 1 + rel * rng.standard_normal(b.shape)
        bins.append(b)
    return fsbm.GridState(s.ranges, s.grid, s.temperature.copy(), s.pressure * (1 + 1e-9), bins)


@pytest.mark.gpu
@pytest.mark.parametrize("rel", [0.0, 1e-3, 1e-7, 1e-13])
def test_compare_states_gpu_equals_reference(reference, rel):
    rng = np.random.default_rng(5)
    a = small_state(seed=11, ni=6, nk=7, nj=9, nkr=33)
    b = _perturbed(a, rng, rel) if rel else a
    rep = fsbm.compare_states(a, b)
    st, ref = reference.compare_states(ranges6(a.ranges), a.grid.x, a.temperature, a.pressure,
                                       np.stack(a.bins), b.grid.x, b.temperature, b.pressure,
                                       np.stack(b.bins))
    assert st == 0
    assert [f.field for f in rep.fields] == ["mass_grid", "temperature", "pressure", "liquid",
                                             "ice1", "ice2", "ice3", "snow", "graupel"]
    for f, (mn, mean, cnt, ex) in zip(rep.fields, ref):
        assert (f.min_digits, f.count_compared, f.count_exact) == (mn, cnt, ex), f.field
        assert f.mean_digits == mean, f.field
    assert rep.all_exact() == (rel == 0.0)
    print(fsbm.format_diff_report(rep))


@pytest.mark.gpu
def test_spec_digit_examples_and_errors(reference):
    # SPEC verify examples: identical -> 16; relative 1e-3 perturbation -> 3
    assert fsbm.digit_agreement(1.25, 1.25) == 16
    assert fsbm.digit_agreement(0.0, -0.0) == 16
    assert fsbm.digit_agreement(2.0, -2.0) == 0
    assert fsbm.digit_agreement(1.0, 1.001) == 3
    for a, b in [(1.0, 1.001), (3.7e-14, 3.7000001e-14), (1e300, 1.0000000000001e300), (5.0, 7.0)]:
        assert fsbm.digit_agreement(a, b) == reference.digit_agreement(a, b)[1]
        assert fsbm.digit_agreement(b, a) == fsbm.digit_agreement(a, b)  # symmetry
    with pytest.raises(fsbm.DomainError, match="finite"):
        fsbm.digit_agreement(float("nan"), 1.0)


@pytest.mark.gpu
def test_compare_fast_vs_exact_step(reference, oracle):
    """The diffwrf use-case: FAST vs EXACT numerics after one step, device states."""
    import torch
    nkr = 33
    grid = fsbm.make_mass_grid(nkr)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry(),
                             fsbm.KernelParams("golovin", 1.0, 1.5, 0.05))
    ctx = fsbm.CoalContext(grid, tabs)
    from paper_2409_07232_b200 import synth
    st, mask = synth.thunderstorm_device(ctx, 6, 8, 20, 0.8, 42)
    out = {}
    for numerics in ("fast", "exact"):
        s2 = fsbm.GridState(st.ranges, grid, st.temperature, st.pressure, [b.clone() for b in st.bins])
        fsbm.fissioned_step(s2, mask, fsbm.StepContext(ctx), fsbm.ExecPlan(numerics=numerics))
        out[numerics] = s2
    rep = fsbm.compare_states(out["fast"], out["exact"])
    h = lambda s: [s.grid.x, s.temperature.cpu().numpy(), s.pressure.cpu().numpy(),
                   torch.stack(s.bins).cpu().numpy()]
    rs, ref = reference.compare_states(ranges6(st.ranges), *h(out["fast"]), *h(out["exact"]))
    assert rs == 0
    for f, (mn, mean, cnt, ex) in zip(rep.fields, ref):
        assert (f.min_digits, f.count_compared, f.count_exact, f.mean_digits) == (mn, cnt, ex, mean)
    assert rep.fields[0].count_exact == nkr and rep.fields[1].count_exact == st.ranges.npoints()
