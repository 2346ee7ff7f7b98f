"""Micro-probe: coarse-level ILU-GMRES(400) per-class device times."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2009_13840_b200 import host, solver as S

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = S.default_context()
mesh = host.Mesh.unit_square(n, tri=True, jitter=0.2, seed=0, neumann="top")
loc = host.LocalSystem(mesh, "hho-dp", "v-cond", 3, data="sincos")
A, b = host.assemble_stokes(loc, ctx=ctx)
t = time.perf_counter()
h = S.LevelHierarchy(A, loc.layout(), S.LevelConfig(degrees=[3, 2, 1, 0], coarse="gmres-ilu"))
print(f"n={n} hierarchy setup {time.perf_counter()-t:.3f} s", flush=True)
m = h.level_matrix(3)
ilu = h.level_ilu(3)
rhs = np.random.default_rng(0).standard_normal(m.n)
S.gmres(m, ilu, rhs, None, 20, 0.0)
ctx.profile(True)
ctx.timer_start()
r = S.gmres(m, ilu, rhs, None, 400, 1e-30)
ms = ctx.timer_stop()
prof = ctx.profile_read()
ctx.profile(False)
print(f"coarse n={m.n}: gmres 400 its {ms:.1f} ms; " + ", ".join(
    f"{k}: {v[0]} x {v[1]/max(v[0],1)*1e3:.1f} us" for k, v in prof.items() if v[0]), flush=True)
