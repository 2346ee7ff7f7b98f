"""Host-side sweep plans (walk.cu) without a GPU: tools/plan_check.cu builds
the forward/backward plans of a pattern and emulates the walkers' data flow
(ring slots, recycled long-range slots, static/far lists, task tables, the
diagonal-major and row-contiguous entry layouts), comparing with the
sequential sweeps of ilu0.hpp:53-65 bit for bit, for every plan variant."""
import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle_ref as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "tools", "plan_check")
SRC = os.path.join(ROOT, "tools", "plan_check.cu")
WALK = os.path.join(ROOT, "paper_2009_13840_b200", "csrc", "walk.cu")

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference oracle not built")


@pytest.fixture(scope="module")
def checker():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    stale = not os.path.exists(CHECK) or any(
        os.path.getmtime(f) > os.path.getmtime(CHECK) for f in (SRC, WALK))
    if stale:
        if not os.path.exists(nvcc):
            pytest.skip("nvcc not available")
        subprocess.run([nvcc, "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-I", os.path.join(ROOT, "include"), "-I",
                        os.path.join(ROOT, "paper_2009_13840_b200", "csrc"), SRC, "-o", CHECK],
                       check=True, capture_output=True)
    return CHECK


CASES = [dict(mesh="unit-tri", n=12, jitter=0.2, seed=0, side="top", scheme="hho-dp",
              strategy="v-cond", k=3, data="sincos"),
         dict(mesh="unit-tri", n=16, jitter=0.2, seed=0, side="top", scheme="hho-dp",
              strategy="v-cond", k=0, data="sincos"),
         dict(family="trapz", n=6, scheme="hho-dp", strategy="vp-cond", k=2),
         dict(family="tri", n=4, scheme="hho-hp", strategy="vp-cond", k=2)]
MODES = [{}, {"PSCU_CHAIN_ROWS": "1"}, {"PSCU_CHAIN_ROWS": "16"},
         {"PSCU_WALK_MODE": "levels"}, {"PSCU_WALK_MODE": "levels", "PSCU_LEVEL_CHAIN_ROWS": "1"},
         {"PSCU_WALK_MODE": "walker", "PSCU_CHAIN_ROWS": "1"},
         {"PSCU_WALK_MODE": "push1", "PSCU_WALK_CLUSTER": "8"}]


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_plans_emulate_bitwise(checker, tmp_path, ci):
    a = O.RefSystem(**CASES[ci]).csr()
    rp, cl = tmp_path / "rp.bin", tmp_path / "c.bin"
    a.row_ptr.astype(np.int64).tofile(rp)
    a.cols.astype(np.int32).tofile(cl)
    for m in MODES:
        env = {k: v for k, v in os.environ.items() if not k.startswith("PSCU_")}
        env.update(m)
        r = subprocess.run([checker, str(rp), str(cl)], capture_output=True, text=True, env=env,
                           timeout=300)
        assert r.returncode == 0, (m, r.stdout, r.stderr)
        assert r.stdout.count("mismatches 0") == 2, (m, r.stdout)


def test_plans_long_rows_fall_back(checker, tmp_path):
    """Rows longer than a walker chunk's diagonal capacity: the push plan is
    reported infeasible and the sweep falls back to task-level launches
    (no exception escapes the planner threads); emulation still bitwise."""
    import synthetic
    a = synthetic.long_row_csr()
    rp, cl = tmp_path / "rp.bin", tmp_path / "c.bin"
    a.row_ptr.astype(np.int64).tofile(rp)
    a.cols.astype(np.int32).tofile(cl)
    for m in MODES[:4]:
        env = {k: v for k, v in os.environ.items() if not k.startswith("PSCU_")}
        env.update(m)
        r = subprocess.run([checker, str(rp), str(cl)], capture_output=True, text=True, env=env,
                           timeout=300)
        assert r.returncode == 0, (m, r.stdout, r.stderr)
        assert r.stdout.count("mismatches 0") == 2, (m, r.stdout)
