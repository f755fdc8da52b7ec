"""GPU: the C++ drop-in (include/pmg_b200/solver.hpp) against the reference's
own pmg::MgSolver / pmg::build_stencils, on cases built by the reference
harness (oracle/cpp_dropin.cpp).  The binary is built in this container by
`make -C oracle dropin` (it needs the reference headers) and travels to the
GPU box in oracle/_ref/."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "cpp_dropin")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="make -C oracle dropin (needs the reference headers)")
def test_cpp_dropin_matches_reference_solver():
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "ALL OK" in p.stdout


HARNESS = os.path.join(ROOT, "oracle", "_ref", "harness_dropin")


@pytest.mark.skipif(not os.path.exists(HARNESS), reason="make -C oracle dropin (needs the reference headers)")
def test_harness_on_gpu_matches_reference_harness():
    """Every case the reference harness knows (harness.hpp:47-54) through
    pmg::b200::run_case and pmg::run_case: residuals.csv, errors.csv,
    mesh_stats.txt, config_resolved.cfg and the dumps agree (oracle/harness_dropin.cpp)."""
    p = subprocess.run([HARNESS], capture_output=True, text=True, timeout=1200)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "ALL OK" in p.stdout
    assert p.stdout.count("\nok ") + p.stdout.startswith("ok ") >= 15
