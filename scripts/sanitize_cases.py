"""One small step per kernel for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck):  python scripts/sanitize_cases.py <case>

cases: dmma (33 bins, headline kernel), dmmag66, dmmag264 (lean layout), direct (coal_fast),
exact, host (pipelined host path), group (two contexts, j-patches), stiff (error path with
the value lock), moments.  Each checks its output against the oracle so a sanitizer run
that perturbs scheduling still has to produce the right numbers."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main(case):
    if case == "direct":
        os.environ["FSBM_FAST_KERNEL"] = "direct"
    import pyoracle
    import torch

    import paper_2409_07232_b200 as fsbm
    from paper_2409_07232_b200 import synth
    from test_gpu_parity import assert_close, make_ctx, run_oracle_grid, thunder_host

    O = pyoracle.Oracle()
    nkr = {"dmmag66": 66, "dmmag264": 264}.get(case, 33)
    dims = {66: (2, 3, 30), 264: (1, 2, 25)}.get(nkr, (3, 4, 40))
    ctx, grid, tabs = make_ctx(nkr, coeff=1500.0 if case == "stiff" else 1.0)
    st, mask, B = thunder_host(O, ctx, *dims, 0.9, 42)
    s, cnt_o, err_o, Bo = run_oracle_grid(O, ctx, tabs, st, mask, B)
    numerics = "exact" if case == "exact" else "fast"
    plan = fsbm.ExecPlan(numerics=numerics)
    if case == "stiff":
        assert s == 4
        with_err = None
        try:
            fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), plan)
        except fsbm.StiffnessError as e:
            with_err = e
        assert with_err is not None and with_err.point == tuple(int(v) for v in err_o[2:5])
        print(f"sanitize case {case}: ok")
        return
    assert s == 0
    if case == "host":
        fsbm.fissioned_step(st, None, fsbm.StepContext(ctx), plan)
        got = np.stack([b.reshape(-1, nkr) for b in st.bins])
    elif case == "group":
        g = fsbm.DeviceGroup(grid, tabs, [0, 0])
        g.step_host(st, None, "j", plan=plan)
        got = np.stack([b.reshape(-1, nkr) for b in st.bins])
        g.close()
    else:
        d = fsbm.GridState(st.ranges, grid, *[torch.from_numpy(np.ascontiguousarray(a)).cuda()
                                              for a in (st.temperature, st.pressure)],
                           [torch.from_numpy(b.copy()).cuda() for b in st.bins])
        if case == "moments":
            import ctypes as C
            from paper_2409_07232_b200 import _lib
            out = (C.c_double * 12)()
            ptrs = (C.c_void_p * 6)(*[b.data_ptr() for b in d.bins])
            _lib.check(_lib.load().fsbm_state_moments_device(ctx.handle, st.ranges.npoints(), ptrs,
                                                             out, None))
            np.testing.assert_allclose(np.array(out[:6]), B.sum(axis=(1, 2)), rtol=1e-13)
            print(f"sanitize case {case}: ok")
            return
        fsbm.fissioned_step(d, None, fsbm.StepContext(ctx), plan)
        got = np.stack([b.cpu().numpy().reshape(-1, nkr) for b in d.bins])
    if numerics == "exact":
        assert np.array_equal(got, Bo)
    else:
        assert_close(got, Bo, case)
    torch.cuda.synchronize()
    print(f"sanitize case {case}: ok ({ctx.fast_kernel() if numerics == 'fast' else 'coal_exact'})")


if __name__ == "__main__":
    main(sys.argv[1])
