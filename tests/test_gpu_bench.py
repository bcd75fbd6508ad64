"""bench.py's own paths on one GPU (small grids): the drop-in path and the device-group path
(FSBM_BENCH_GROUP=1: the N>1 code as a one-rank group) report the same counts, a green
parity block and a JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(extra_env=None, *args):
    env = dict(os.environ)
    env.update(extra_env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--ni", "12", "--steps", "2",
                          "--warmup", "1", "--no-e2e", "--no-exact", "--no-configs", "--cpu-seconds", "1",
                          *args], capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_bench_line_contract_and_group_path():
    a = run_bench()
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "dtype", "config", "roofline", "cpu_baseline", "parity", "clocks", "gpu_launches"):
        assert k in a, k
    assert a["parity"]["green"] and a["parity"]["counters_equal"]
    assert a["gpu_launches"] > 0 and a["value"] > 0
    b = run_bench({"FSBM_BENCH_GROUP": "1"})
    assert b["diagnostics"]["updates_per_step"] == a["diagnostics"]["updates_per_step"]
    assert b["diagnostics"]["triples_per_step"] == a["diagnostics"]["triples_per_step"]
    assert abs(b["diagnostics"]["mass_after"] - a["diagnostics"]["mass_after"]) <= 1e-12 * a["diagnostics"]["mass_after"]
