"""In-tree build of the sm_100a solver library and (for tests) the oracles.

``build_native()`` compiles paper_2009_13840_b200/csrc/*.cu with nvcc for
``-gencode arch=compute_100a,code=sm_100a`` into
paper_2009_13840_b200/libpstokes_b200.so (git-ignored, travels to the GPU
box with the gpurun snapshot). ``--fmad=false`` and ``-ffp-contract=off``
keep every floating-point operation individually rounded so the device
results are bit-identical to the reference's operation order.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libpstokes_b200.so")
HOST_LIB = os.path.join(PKG, "libpstokes_host.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off", "-Wno-deprecated-gpu-targets",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build the solver")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_native(force: bool = False, verbose: bool = False, trace: bool = False,
                 variant: str = "", defines=()) -> str:
    """Builds libpstokes_b200.so. trace=True builds the walker-instrumented
    variant (-DPSCU_TRACE; PSCU_WALK_TRACE=1 at run time) into
    tools/libpstokes_trace.so instead (diagnostics: PSCU_LIB=<that path>)."""
    nvcc = _nvcc()
    obj_dir = os.path.join(PKG, "_build_trace") if trace else OBJ
    lib = os.path.join(ROOT, "tools", "libpstokes_trace.so") if trace else LIB
    flags = NVCC_FLAGS + (["-DPSCU_TRACE"] if trace else [])
    if variant:
        # tuning builds (compile-time knobs): tools/libpstokes_<variant>.so, PSCU_LIB=<that path>
        obj_dir = os.path.join(PKG, "_build_" + variant)
        lib = os.path.join(ROOT, "tools", f"libpstokes_{variant}.so")
        flags = flags + ["-D" + d for d in defines]
    os.makedirs(obj_dir, exist_ok=True)
    sources = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "pstokes_cuda.h"))
    jobs = []
    objs = []
    for src in sources:
        s = os.path.join(CSRC, src)
        o = os.path.join(obj_dir, src[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([nvcc, *flags, "-c", s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {cmd[-3]}:\n{r.stderr}")

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib, objs):
        run([nvcc, "-shared", "-o", lib, *objs, "-lcudart"])
    return lib


def build_host(force: bool = False) -> str:
    """Host-side input producer (mesh, bases, HHO local blocks, pattern)."""
    src_dir = os.path.join(PKG, "host")
    if not os.path.isdir(src_dir):
        return ""
    sources = sorted(os.path.join(src_dir, f) for f in os.listdir(src_dir) if f.endswith(".cpp"))
    headers = [os.path.join(src_dir, f) for f in os.listdir(src_dir) if f.endswith(".hpp")]
    if not sources:
        return ""
    if force or _stale(HOST_LIB, sources + headers):
        cmd = ["g++", "-std=c++20", "-O3", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-I" + os.path.join(ROOT, "include"), "-I" + src_dir, "-o", HOST_LIB, *sources]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"host build failed:\n{r.stderr}")
    return HOST_LIB


def build_oracle(force: bool = False) -> None:
    """Builds oracle/_build (C restatement) and, when /root/reference is
    present, oracle/_ref (the reference compiled in place). Test
    infrastructure only."""
    oracle = os.path.join(ROOT, "oracle")
    targets = ["restatement"]
    if os.path.isdir("/root/reference/proj/include"):
        targets.append(os.path.join(oracle, "_ref", "libpstokes_ref.so"))
        targets.append(os.path.join(oracle, "_ref", "wire_ref"))
        if os.path.exists(LIB):
            targets.append("dropin")  # links the solver library
    cmd = ["make", "-C", oracle, *targets]
    if force:
        cmd.insert(1, "-B")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


if __name__ == "__main__":
    f = "--force" in sys.argv
    print(build_native(force=f, verbose=True))
    print(build_host(force=f))
    build_oracle(force=f)
