"""The compiled C++ drop-in (integration/gpu_fissioned_step.cpp, coalbench::fissioned_step's
signature) against the unmodified reference in one binary (integration/test_dropin.cpp):
EXACT bitwise, FAST within the bar, identical exception types / points / messages."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "integration", "_build", "test_dropin")


def test_cpp_dropin_matches_reference_fissioned_step():
    if not os.path.exists(EXE):
        if not os.path.isdir("/root/reference/proj/src"):
            pytest.skip("integration/_build/test_dropin not built (needs the reference sources; "
                        "__graft_entry__.build() makes it)")
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "integration")], check=True)
    out = subprocess.run([EXE], capture_output=True, text=True, timeout=900)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "dropin ok" in out.stdout
