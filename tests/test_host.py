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
