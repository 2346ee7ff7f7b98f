"""Micro-probe: device-timed ILU(0) applies / SpMVs per level matrix."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2009_13840_b200 import host, solver as S, _native as N

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ctx = S.default_context()
mesh = host.Mesh.unit_square(n, tri=True, jitter=0.2, seed=0, neumann="top")
loc = host.LocalSystem(mesh, "hho-dp", "v-cond", 3, data="sincos")
A, b = host.assemble_stokes(loc, ctx=ctx)
t = time.perf_counter()
h = S.LevelHierarchy(A, loc.layout(), S.LevelConfig(degrees=[3, 2, 1, 0], coarse="gmres-ilu"))
print(f"hierarchy setup {time.perf_counter()-t:.3f} s", flush=True)
lib = ctx.lib
levels = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else range(4)
for l in levels:
    ilu = h.level_ilu(l)
    m = h.level_matrix(l)
    x = torch.randn(m.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    N.check(lib.pscu_ilu0_apply(ctx.h, ilu.h, x.data_ptr(), y.data_ptr(), N.PSCU_DEVICE))
    ctx.timer_start()
    for _ in range(reps):
        N.check(lib.pscu_ilu0_apply(ctx.h, ilu.h, x.data_ptr(), y.data_ptr(), N.PSCU_DEVICE))
    ms = ctx.timer_stop() / reps
    ctx.timer_start()
    for _ in range(reps):
        N.check(lib.pscu_spmv(ctx.h, m.h, x.data_ptr(), y.data_ptr(), N.PSCU_DEVICE))
    ms2 = ctx.timer_stop() / reps
    print(f"level {l}: n={m.n} nnz={m.nnz} ilu apply {ms:.3f} ms   spmv {ms2*1e3:.1f} us "
          f"({(12*m.nnz+16*m.n)/ms2/1e6:.0f} GB/s incl. indices)", flush=True)
