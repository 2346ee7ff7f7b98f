#!/usr/bin/env python
"""Generates tests/golden/c2_<variant>_<n>.json: reference solves of the
BASELINE.json config-2 recipe (unit square, n x n cells split into
triangles, 0.2h jitter with SplitMix64(0), HHO-dp k=3, levels 3-2-1-0,
V(2,2) ILU(0)-GMRES smoother, ILU-GMRES coarse (1e-3, 400), FGMRES(30) to
rtol 1e-8, sin/cos data) run by the UNMODIFIED reference (oracle/_ref,
plevels.hpp:217-239 through ref_driver.cpp's fgmres_hist).

Each fixture stores the integer counts (FGMRES its, coarse its, V-cycles),
the full residual history, the relative residual, sampled solution entries
plus a SHA-256 of the whole solution and of the assembled operator, and the
reference's own t_solve on this container's core (one thread).

Usage: python tools/gen_c2_fixtures.py v-cond 64 [v-cond 128 ...]
Test infrastructure: run here (needs /root/reference for oracle/_ref).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_ref as O  # noqa: E402

SAMPLE_STRIDE = 997


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run(strategy: str, n: int) -> dict:
    t0 = time.time()
    s = O.RefSystem(mesh="unit-tri", n=n, seed=0, jitter=0.2, side="top", scheme="hho-dp",
                    strategy=strategy, k=3, data="sincos")
    a = s.csr()
    b = s.rhs()
    t_asm = time.time() - t0
    r = s.solve([3, 2, 1, 0], coarse="gmres-ilu", rtol=1e-8, restart=30, maxit=1000)
    x = r["x"]
    idx = np.arange(0, len(x), SAMPLE_STRIDE, dtype=np.int64)
    return {
        "recipe": f"unit-tri n={n} jitter=0.2 seed=0 hho-dp {strategy} k=3 levels 3-2-1-0 "
                  "V(2,2) ILU(0)-GMRES smoother, ILU-GMRES coarse 1e-3/400, FGMRES(30) rtol 1e-8, "
                  "sincos data, Neumann top",
        "generator": "tools/gen_c2_fixtures.py (oracle/_ref = unmodified reference headers)",
        "n_cells": n, "strategy": strategy, "dim": int(a.n), "nnz": int(a.nnz),
        "operator_sha256": digest(a.row_ptr, a.cols, a.vals),
        "rhs_sha256": digest(b),
        "its": r["its"], "coarse_its": int(r["coarse_its"]), "vcycles": r["vcycles"],
        "converged": r["converged"], "rel": r["rel"],
        "hist": [float(v) for v in r["hist"]],
        "x_sha256": digest(x), "x_norm2": float(np.sqrt(np.dot(x, x))),
        "x_maxabs": float(np.max(np.abs(x))),
        "x_sample_stride": SAMPLE_STRIDE, "x_sample": [float(v) for v in x[idx]],
        "t_solve_ref_s": r["t_solve"], "t_assembly_s": t_asm, "cores": 1,
    }


def main():
    args = sys.argv[1:]
    out_dir = os.path.join(ROOT, "tests", "golden")
    for strategy, n in zip(args[::2], args[1::2]):
        d = run(strategy, int(n))
        name = f"c2_{strategy.replace('-', '')}_{n}.json"
        with open(os.path.join(out_dir, name), "w") as f:
            json.dump(d, f, indent=1)
        print(name, d["its"], d["coarse_its"], d["vcycles"], f"{d['t_solve_ref_s']:.1f}s",
              flush=True)


if __name__ == "__main__":
    main()
