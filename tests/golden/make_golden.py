"""Generate tests/golden/*.npz from the REAL reference (oracle/_ref/libcoalbench_ref.so).

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle  # noqa: E402

pyoracle.build(ref=True)
R = pyoracle.Reference()
O = pyoracle.Oracle()


def thunder_bins(nkr, ratio, seed, npts):
    x = R.mass_grid(nkr, 3.35e-14, ratio)
    return np.stack([O.thunderstorm_point(x, seed, p) for p in range(npts)])  # (npts, 6, nkr)


def main():
    out = {}
    # 1. SPEC hand oracles through the real coal_step
    for name, x, nb, init in (("two_bin", [1.0, 2.0], 2, [2.0, 0.0]),
                              ("three_bin", [1.0, 2.0, 4.0], 3, [0.0, 1.0, 0.0])):
        ratio = 2.0
        abd = np.array([0, 0, 0], np.int32)
        t750, t500 = R.build_tables(nb, x1=1.0, ratio=ratio, abd=abd, family=0, coeff=1.0,
                                    level_scale=1.0)
        b = np.zeros((6, nb))
        b[0] = init
        st, cnt, _ = R.coal_step(nb, t750, t500, b, 600.0, dt=0.1, x1=1.0, ratio=ratio, abd=abd)
        assert st == 0
        out[f"hand_{name}_in"] = np.array(init)
        out[f"hand_{name}_out"] = b[0].copy()
        out[f"hand_{name}_counters"] = cnt
    # 2. per-point coal_step on thunderstorm spectra, nkr in {17, 33, 66}, 2 pressures
    for nkr in (17, 33, 66):
        ratio = pyoracle.equal_range_ratio(nkr)
        t750, t500 = R.build_tables(nkr, ratio=ratio, pair_scale_step=0.05)
        pts = thunder_bins(nkr, ratio, 42, 4)
        outs, cnts = [], []
        for q, pres in enumerate((900.0, 625.0, 612.5, 400.0)):
            b = pts[q].copy()
            st, cnt, _ = R.coal_step(nkr, t750, t500, b, pres, dt=1.0, substeps=2 if q == 1 else 1,
                                     ratio=ratio)
            assert st == 0
            outs.append(b)
            cnts.append(cnt)
        out[f"point_nkr{nkr}_in"] = pts
        out[f"point_nkr{nkr}_out"] = np.stack(outs)
        out[f"point_nkr{nkr}_counters"] = np.stack(cnts)
        out[f"point_nkr{nkr}_pressure"] = np.array([900.0, 625.0, 612.5, 400.0])
        lo, wlo, whi, top = R.gain_table(nkr, ratio=ratio)
        out[f"gain_nkr{nkr}_lo"] = lo
        out[f"gain_nkr{nkr}_wlo"] = wlo
        out[f"gain_nkr{nkr}_whi"] = whi
        out[f"gain_nkr{nkr}_top"] = top
    # 3. a small fissioned_step on make_synthetic_case (liquid only), 4x5x6, cf 0.3, seed 42
    ni, nk, nj, nkr = 4, 5, 6, 33
    T, P, bins = R.synthetic_case(ni, nk, nj, 0.3, 42, nkr)
    t750, t500 = R.build_tables(nkr, pair_scale_step=0.05)
    b = bins.copy()
    st, cnt, _, err = R.fissioned_step(ni, nk, nj, nkr, t750, t500, T, P, b, threads=2)
    assert st == 0
    out["grid_T"], out["grid_P"], out["grid_in"], out["grid_out"] = T, P, bins, b
    out["grid_counters"] = cnt
    # 4. mask count example: 10x10x10, cf 0.3, seed 42 -> 300
    T, P, _ = R.synthetic_case(10, 10, 10, 0.3, 42, 33)
    mask, cnt = R.fission_predicates(10, 10, 10, T)
    out["mask_10cube_count"] = np.array(cnt)
    out["mask_10cube"] = mask
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
