"""Host-side logic and the C-ABI boundary, CPU only (no compute calls)."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import paper_2409_07232_b200 as fsbm
from paper_2409_07232_b200 import _lib, synth


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _lib.header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True,
                         text=True).stdout
    for s in syms:
        assert f" T {s}" in out, f"{s} not exported"


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    grid = fsbm.make_mass_grid(33)
    tabs = fsbm.build_tables(grid, fsbm.default_pair_registry())
    with pytest.raises(fsbm.CudaError):
        fsbm.CoalContext(grid, tabs)


def test_mass_grid_and_tables_match_reference(reference):
    for nkr in (17, 33, 66):
        r = fsbm.equal_range_ratio(nkr)
        g = fsbm.make_mass_grid(nkr, 3.35e-14, r)
        assert np.array_equal(g.x, reference.mass_grid(nkr, 3.35e-14, r))
        for fam, fid in (("golovin", 1), ("constant", 0), ("product", 2)):
            t = fsbm.build_tables(g, fsbm.default_pair_registry(),
                                  fsbm.KernelParams(fam, 0.9, 1.5, 0.05))
            a, b = reference.build_tables(nkr, ratio=r, family=fid, coeff=0.9, pair_scale_step=0.05)
            assert np.array_equal(t.t750.reshape(-1), a) and np.array_equal(t.t500.reshape(-1), b)


def test_registry_matches_reference(reference):
    abd = np.array([[p.source_a, p.source_b, p.dest] for p in fsbm.default_pair_registry()],
                   np.int32).reshape(-1)
    assert np.array_equal(abd, reference.default_registry())
    with pytest.raises(fsbm.ConfigError):
        fsbm.validate_registry(fsbm.default_pair_registry()[:19])


def test_synth_thermo_matches_make_synthetic_case(reference):
    grid = fsbm.make_mass_grid(33)
    for cf, seed in ((0.3, 42), (1.0, 1), (0.0, 7)):
        T, P, liq = synth.thermo_host(7, 6, 5, cf, seed, grid, liquid=True)
        T2, P2, B2 = reference.synthetic_case(7, 6, 5, cf, seed, 33)
        assert np.array_equal(T, T2) and np.array_equal(P, P2)
        assert np.array_equal(liq, B2[0].reshape(-1))


def test_decompose_matches_reference_semantics():
    r = fsbm.Ranges(1, 8, 1, 3, 1, 8)
    assert fsbm.decompose(r, 1, 1).tiles == [(1, 8, 1, 8)]
    assert fsbm.decompose(r, 2, 2).tiles == [(1, 4, 1, 4), (5, 8, 1, 4), (1, 4, 5, 8), (5, 8, 5, 8)]
    with pytest.raises(fsbm.DomainError):
        fsbm.decompose(fsbm.Ranges(1, 5, 1, 1, 1, 1), 2, 1)


def test_plan_validation_host_side():
    with pytest.raises(fsbm.ConfigError):
        fsbm.ExecPlan(numerics="bogus").to_c()
    p = fsbm.ExecPlan(mode="parallel", collapse=3, threads=8, scratch_strategy="arena").to_c()
    assert (p.collapse, p.threads, p.scratch_strategy) == (3, 8, 1)


def test_pressure_weight_and_interp():
    assert fsbm.pressure_weight(625.0) == 0.5
    assert fsbm.interpolate_kernel(3.0, 4.5, 0.5) == 3.75
    assert fsbm.pressure_weight(100.0) == 0.0 and fsbm.pressure_weight(1000.0) == 1.0


def test_decompose_shards_match_reference_decompose():
    """fsbm_decompose (C ABI) == decompose's split_range (driver.cpp:35-51,187-196)."""
    from paper_2409_07232_b200 import shard
    r = fsbm.Ranges(1, 425, 1, 50, 1, 300)
    for n in (1, 2, 3, 4, 8, 7):
        jp = shard.decompose_shards(r, n, "j")
        ref = fsbm.decompose(r, n, 1).tiles  # (its, ite, jts, jte), one tile per patch
        assert [(p.jds, p.jde) for p in jp] == [(t[2], t[3]) for t in ref]
        assert all((p.ids, p.ide, p.kds, p.kde) == (1, 425, 1, 50) for p in jp)
        ip = shard.decompose_shards(r, n, "i")
        ref = fsbm.decompose(r, 1, n).tiles
        assert [(p.ids, p.ide) for p in ip] == [(t[0], t[1]) for t in ref]
    with pytest.raises(fsbm.DomainError):
        shard.decompose_shards(fsbm.Ranges(1, 3, 1, 1, 1, 2), 3, "j")
    with pytest.raises(fsbm.ConfigError):
        _lib.check(_lib.load().fsbm_decompose(r.to_c(), 2, 5, (_lib.fsbm_ranges * 2)()))


def test_fissioned_step_validates_buffers():
    """dtype / size / contiguity / placement are checked before any raw pointer
    reaches the C ABI (ShapeError / DomainError, no out-of-bounds access)."""
    grid = fsbm.make_mass_grid(33)
    r = fsbm.Ranges(1, 2, 1, 2, 1, 2)
    n = r.npoints()
    good = lambda: [np.zeros(n * 33) for _ in range(6)]
    T, P = np.full(n, 250.0), np.full(n, 600.0)

    class _Ctx:  # validation runs before any library call
        nkr, device = 33, 0
    sctx = fsbm.StepContext(_Ctx())
    cases = [
        (fsbm.GridState(r, grid, T, P, [b.astype(np.float32) for b in good()]), None, fsbm.ShapeError),
        (fsbm.GridState(r, grid, T, P, [np.zeros(n * 33 - 1)] + good()[1:]), None, fsbm.ShapeError),
        (fsbm.GridState(r, grid, T, P[:-1], good()), None, fsbm.ShapeError),
        (fsbm.GridState(r, grid, T, P, [np.zeros((n * 33, 2))[:, 0]] + good()[1:]), None, fsbm.ShapeError),
        (fsbm.GridState(r, grid, T, P, good()), fsbm.PredicateMask(r, np.zeros(n, np.int32)), fsbm.ShapeError),
        (fsbm.GridState(r, grid, T, None, good()), None, fsbm.DomainError),
        (fsbm.GridState(r, grid, T, P, good()[:5]), None, fsbm.ShapeError),
    ]
    for st, m, exc in cases:
        with pytest.raises(exc):
            fsbm.fissioned_step(st, m, sctx, fsbm.ExecPlan())


def test_bench_reference_arm_never_loads_the_product(tmp_path):
    """The reference arm (bench.py --impl reference) runs oracle/_ref on inputs from the
    checkers only: no paper_2409_07232_b200 import, no libfsbm_coal.so mapping."""
    import json
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, runpy; sys.argv = ['bench.py', '--impl', 'reference', '--ni', '3', "
            "'--nj', '8', '--nk', '5', '--steps', '1', '--warmup', '1']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT', any(m.startswith('paper_2409') for m in sys.modules), "
            "'libfsbm_coal' in maps)")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[-2])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    assert lines[-1] == "PRODUCT False False"
