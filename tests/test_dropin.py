"""The C++ drop-in layer (include/pstokes_b200/pstokes_b200.hpp) next to the
reference's own code path: tests/cpp/dropin_driver.cpp, compiled against the
unmodified reference headers by oracle/Makefile (target dropin), runs
pstokes::solve_system and pstokes::b200::solve_system on the same system,
the reference's fgmres over the device V-cycle (ApplyFn adapters) and the
reference's gmres over device SpMV / ILU(0); every check is bitwise."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "dropin_driver")
HEADER = os.path.join(ROOT, "include", "pstokes_b200", "pstokes_b200.hpp")


def test_header_declares_reference_signatures():
    src = open(HEADER).read()
    for sym in ("solve_system(const Mesh&, const StokesSystem& sys, const LevelConfig& cfg)",
                "class DeviceCsr", "class DeviceIlu0", "class DeviceHierarchy", "ApplyFn apply_fn",
                "ApplyFn vcycle_fn", "pscu_solve_system", "std::invalid_argument"):
        assert sym in src, sym


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DRIVER), reason="drop-in driver not built (needs the reference)")
def test_dropin_driver_bitwise():
    r = subprocess.run([DRIVER], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin: all checks passed" in r.stdout
