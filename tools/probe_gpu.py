"""Scratch GPU probe: times the device solver on oracle-assembled systems."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle_ref as O
from paper_2009_13840_b200 import solver as S

def lay(s):
    L = s.layout
    return S.make_layout(L.scheme, L.strategy, L.k, L.n_faces, L.n_elements)

def timeit(f, reps=5):
    f(); t = time.perf_counter()
    for _ in range(reps): f()
    return (time.perf_counter() - t) / reps

for n in [int(v) for v in (sys.argv[1:] or ["32", "64"])]:
    t = time.time()
    s = O.RefSystem(mesh="unit-tri", n=n, seed=0, jitter=0.2, side="top", k=3, data="sincos")
    a = s.csr(); b = s.rhs()
    print(f"n={n} dim={a.n} nnz={a.nnz} assemble(ref cpu)={time.time()-t:.1f}s", flush=True)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    x = np.random.default_rng(0).standard_normal(a.n)
    print(f"  spmv host-api {timeit(lambda: m.multiply(x))*1e3:.3f} ms", flush=True)
    t = time.time(); ilu = S.Ilu0(m); print(f"  ilu0 factor {time.time()-t:.3f} s", flush=True)
    print(f"  ilu apply host-api {timeit(lambda: ilu.apply(x))*1e3:.3f} ms", flush=True)
    cfg = S.LevelConfig(degrees=[3, 2, 1, 0], coarse="gmres-ilu", outer_rtol=1e-8)
    t = time.time(); h = S.LevelHierarchy(m, lay(s), cfg); ts = time.time() - t
    print(f"  hierarchy setup {ts:.3f} s", flush=True)
    t = time.time(); xs, hist, rep = h.solve(b); tsol = time.time() - t
    print(f"  solve {tsol:.3f} s its={rep.outer_its} coarse_its={rep.coarse_its} rel={rep.rel_residual:.3e} conv={rep.converged}", flush=True)
    print(f"  DoF/s (setup+solve) = {a.n/(ts+tsol):.3e}", flush=True)
