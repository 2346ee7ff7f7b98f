#!/usr/bin/env python
"""3D HHO-hp solve timing on one GPU (diagnostics for configs 3 / 5):
host local blocks -> streamed device condensation + face-block assembly ->
hierarchy + FGMRES. Prints phase times, iteration counts and the per-class
device profile. Usage: python tools/run3d.py N [jitter seed fseed]."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2009_13840_b200 import host  # noqa: E402
from paper_2009_13840_b200 import solver as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
jit = float(sys.argv[2]) if len(sys.argv) > 2 else 0.15
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 1
fseed = int(sys.argv[4]) if len(sys.argv) > 4 else 2
smooth = int(os.environ.get("SMOOTH", "3"))
ctx = S.default_context()
t0 = time.time()
mesh = host.Mesh3(n, jitter=jit, seed=seed)
t1 = time.time()
A, b, lay, info = host.assemble_stokes3(mesh, 2, data="random", seed=fseed, ctx=ctx)
t2 = time.time()
print(f"n={n} faces={mesh.n_faces} dofs={A.n} nnz={A.nnz} mesh {t1-t0:.2f}s assemble {t2-t1:.2f}s "
      f"(local {info['t_local_s']:.2f}s, device {info['t_condense_s']:.2f}s)", flush=True)
cfg = S.LevelConfig(degrees=[2, 1, 0], smoother_iters=smooth, coarse="gmres-ilu",
                    smoother="bjacobi", outer_rtol=1e-8, restart=30)
# VARIANTS="K=V K2=V2;K=V3 ...": one solve per variant (plan-time env knobs),
# after REPS plain repetitions
variants = [v.split() for v in os.environ.get("VARIANTS", "").split(";") if v.strip()]
runs = [[]] * int(os.environ.get("REPS", "2")) + variants
for var in runs:
    for kv in var:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    ctx.profile(True)
    ctx.timer_start()
    h = S.LevelHierarchy(A, lay, cfg)
    t_setup = ctx.timer_stop()
    ctx.timer_start()
    x, hist, rep = h.solve(b)
    t_solve = ctx.timer_stop()
    prof = ctx.profile_read()
    ctx.profile(False)
    del h
    print(json.dumps(dict(variant=" ".join(var), setup_ms=t_setup, solve_ms=t_solve, its=rep.outer_its,
                          coarse_its=rep.coarse_its, vcycles=rep.vcycles,
                          rel=rep.rel_residual, conv=rep.converged,
                          dofs_per_s=A.n / ((t_setup + t_solve) / 1e3),
                          classes={k: dict(n=v[0], ms=round(v[1], 2),
                                           GBps=round(v[2] / max(v[1], 1e-9) / 1e6, 1))
                                   for k, v in prof.items()})), flush=True)
