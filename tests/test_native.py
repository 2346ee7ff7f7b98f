"""CPU checks of the drop-in boundary: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/pstokes_cuda.h declares. No compute
call is made here (no GPU in this container)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2009_13840_b200 import _native, build

ROOT = build.ROOT
HEADER = os.path.join(ROOT, "include", "pstokes_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pscu_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_for_sm100a():
    lib = build.build_native()
    assert os.path.exists(lib)
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(build.build_native())
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.EXPORTS) == syms


def test_no_device_fails_loudly():
    """Without a GPU the context creation must fail (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2009_13840_b200 import solver

    with pytest.raises(Exception):
        solver.Context(0)


def test_device_list_create_fails_loudly_without_gpu():
    """pscu_create_devices (SURVEY §8(b) signature): bad lists are rejected,
    and without a GPU it fails like pscu_create, leaving no context behind."""
    import torch

    lib = _native.load()
    out = (ctypes.c_void_p * 2)()
    assert lib.pscu_create_devices(None, 0, out) != 0
    devs = (ctypes.c_int32 * 2)(0, 0)
    assert lib.pscu_create_devices(devs, 2, out) != 0  # listed twice, or no device
    assert out[0] is None and out[1] is None
    if not torch.cuda.is_available():
        one = (ctypes.c_int32 * 1)(0)
        assert lib.pscu_create_devices(one, 1, out) != 0
        assert out[0] is None
        assert b"device" in lib.pscu_last_error().lower()


def test_host_library_exports_every_declared_symbol():
    """include/pstokes_host.h (the 2D and 3D host producers) likewise."""
    text = open(os.path.join(ROOT, "include", "pstokes_host.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    syms = sorted(set(re.findall(r"\b(psh3?_[a-z0-9_]+)\s*\(", text)))
    assert "psh_error_tables" in syms and "psh3_local_blocks" in syms
    lib = ctypes.CDLL(build.build_host())
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
