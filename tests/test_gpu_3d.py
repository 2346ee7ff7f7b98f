"""GPU parity of the 3D HHO-hp path (BASELINE.json configs 3 and 5) against
the oracle restatement on identical host-built local blocks
(host/pstokes_host3d.cpp): streamed device condensation + face-block
assembly, the face-block SpMV, p-level inheritance, block-Jacobi smoothing,
V-cycles and full FGMRES solves. The 3D path has no reference (the
reference is 2D only); the oracle is oracle/pstokes_oracle.c's
restatement of the reference's algorithms in 3D. Bar: bitwise (IEEE ==)."""
import numpy as np
import pytest

import oracle_ref as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.port_available(),
                                                  reason="oracle restatement not built")]


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.fixture(scope="module")
def M():
    from paper_2009_13840_b200 import build, host, solver
    build.build_host()
    return host, solver


def _oracle_system(host, n, jitter, data, k=2, seed=2):
    m = host.Mesh3(n, jitter=jitter, seed=1)
    L = host.HpLocal3(k)
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data=data, seed=seed)
    brp, bcols = m.block_pattern()
    rp, cols = O.bsr_to_csr_pattern(brp, bcols, L.face_block)
    lay = O.po_layout(1, 2, k, m.n_faces, m.n_elements, dim=3)
    a, b = O.port_condense_assemble(mats, rhs, L.n_local, L.elim, L.kept_global(m.element_faces()),
                                    lay, rp, cols)
    return m, L, mats, rhs, brp, bcols, a, b, lay


@pytest.mark.parametrize("n,jitter,batch", [(2, 0.0, 3), (3, 0.15, 7), (4, 0.15, 4096)])
def test_streamed_assembly_bitwise(M, n, jitter, batch):
    host, S = M
    m, L, mats, rhs, brp, bcols, a, b, lay = _oracle_system(host, n, jitter, "random")
    A, bd, lay_d, info = host.assemble_stokes3(m, 2, data="random", seed=2, batch=batch)
    rp, cl, vl = A.download()
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(cl, a.cols)
    assert same(vl, a.vals)
    assert same(bd, b)
    assert S.layout_dim(lay_d) == a.n


def test_recovery_data_bitwise(M):
    host, S = M
    m = host.Mesh3(2, jitter=0.1, seed=1)
    L = host.HpLocal3(2)
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data="random", seed=5)
    A, b, lay, info = host.assemble_stokes3(m, 2, data="random", seed=5, batch=3, recovery=True)
    lib = O.port_lib()
    n, ne, nk = L.n_local, L.n_elim, L.n_keep
    for e in range(m.n_elements):
        sch, rr = np.zeros(nk * nk), np.zeros(nk)
        cp, er = np.zeros(ne * nk), np.zeros(ne)
        el = np.ascontiguousarray(L.elim, np.int32)
        assert lib.po_condense(n, mats[e * n * n:(e + 1) * n * n].copy(), rhs[e * n:(e + 1) * n].copy(),
                               ne, el, sch, rr, cp, er) == 0
        assert same(info["elim_coupling"][e], cp.reshape(nk, ne).T)
        assert same(info["elim_rhs"][e], er)


def test_bsr_spmv_bitwise(M):
    host, S = M
    m, L, mats, rhs, brp, bcols, a, b, lay = _oracle_system(host, 4, 0.15, "random")
    bv = S.csr_to_bsr_values(a.row_ptr, a.cols, a.vals, brp, bcols, L.face_block)
    A = S.bsr_matrix(brp, bcols, bv, L.face_block)
    lib = O.port_lib()
    pa = O.po_csr(a)
    import ctypes as C
    for seed in range(3):
        x = np.random.default_rng(seed).standard_normal(a.n)
        y = np.zeros(a.n)
        lib.po_csr_multiply(C.byref(pa), x, y)
        assert same(A.multiply(x), y)


@pytest.mark.parametrize("n,jitter,data", [(3, 0.15, "random"), (4, 0.15, "manufactured")])
def test_hierarchy_vcycle_and_solve_bitwise(M, n, jitter, data):
    """Levels 2 -> 1 -> 0, block-Jacobi-preconditioned GMRES(2) smoothing on
    the face-block levels, ILU-GMRES on the coarsest (CSR) level, FGMRES(30)
    to 1e-8: inherited operators, a V-cycle, ITs and the whole residual
    history and solution bit for bit against the oracle."""
    host, S = M
    m, L, mats, rhs, brp, bcols, a, b, lay = _oracle_system(host, n, jitter, data)
    A, bd, lay_d, info = host.assemble_stokes3(m, 2, data=data, seed=2)
    ref = O.PortHierarchy(a, lay, [2, 1, 0], smoother_iters=2, smoother=1)
    cfg = S.LevelConfig(degrees=[2, 1, 0], coarse="gmres-ilu", smoother="bjacobi",
                        outer_rtol=1e-8, restart=30)
    h = S.LevelHierarchy(A, lay_d, cfg)
    for l in range(3):
        rp, cl, vl = h.level_matrix(l).download()
        r = ref.level_csr(l)
        assert np.array_equal(rp, r.row_ptr) and np.array_equal(cl, r.cols) and same(vl, r.vals), l
    d = np.random.default_rng(4).standard_normal(a.n)
    assert same(h.vcycle(0, d), ref.vcycle(0, d))
    r = ref.solve(b, rtol=1e-8, maxit=200, restart=30)
    x, hist, rep = h.solve(bd)
    assert rep.converged and r["converged"]
    assert rep.outer_its == r["its"] and rep.coarse_its == r["coarse_its"]
    assert same(hist, r["hist"]) and same(x, r["x"])
    # one-call drop-in entry on host buffers
    bv = S.csr_to_bsr_values(a.row_ptr, a.cols, a.vals, brp, bcols, L.face_block)
    x2, hist2, rep2 = S.solve_system_bsr(brp, bcols, bv, L.face_block, b, lay_d, cfg)
    assert rep2.outer_its == r["its"] and same(x2, r["x"]) and same(hist2, r["hist"])


def test_bjacobi_face_blocks_bitwise(M):
    host, S = M
    m, L, mats, rhs, brp, bcols, a, b, lay = _oracle_system(host, 3, 0.15, "random")
    A, bd, lay_d, info = host.assemble_stokes3(m, 2, data="random", seed=2)
    bj = S.BlockJacobi(A, lay_d)
    ref = O.PortBlockJacobi(a, lay)
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert same(bj.apply(x), ref.apply(x))


def test_inherit_bsr_matches_csr(M):
    """pscu_inherit on block storage equals inherit_matrix on the CSR
    expansion (plevels.hpp:93-113), for both coarse degrees."""
    host, S = M
    m, L, mats, rhs, brp, bcols, a, b, lay = _oracle_system(host, 3, 0.1, "random")
    bv = S.csr_to_bsr_values(a.row_ptr, a.cols, a.vals, brp, bcols, L.face_block)
    A = S.bsr_matrix(brp, bcols, bv, L.face_block)
    Ac = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    lf = S.make_layout3(2, m.n_faces, m.n_elements)
    for kc in (1, 0):
        lc = S.make_layout3(kc, m.n_faces, m.n_elements)
        r1 = S.inherit_matrix(A, lf, lc).download()
        r2 = S.inherit_matrix(Ac, lf, lc).download()
        assert all(np.array_equal(u, v) for u, v in zip(r1, r2))


def test_dmma_condensation_variant_within_tolerance(M, monkeypatch):
    """PSCU_CONDENSE_DMMA=1: the Schur products A_ke X on the FP64 tensor pipe
    (mma.sync.m8n8k4.f64). The tensor pipe fuses each multiply-add, so the
    operator agrees with the reference-order (bitwise) path to rounding, not
    bit for bit; the bar is BASELINE.json's: same pattern and iteration
    counts, residual history and solution within 1e-9 relative."""
    host, S = M
    m = host.Mesh3(4, jitter=0.15, seed=1)
    A0, b0, lay, _ = host.assemble_stokes3(m, 2, data="random", seed=2)
    monkeypatch.setenv("PSCU_CONDENSE_DMMA", "1")
    A1, b1, lay1, _ = host.assemble_stokes3(m, 2, data="random", seed=2, batch=37)
    monkeypatch.delenv("PSCU_CONDENSE_DMMA")
    rp0, c0, v0 = A0.download()
    rp1, c1, v1 = A1.download()
    assert np.array_equal(rp0, rp1) and np.array_equal(c0, c1)
    scale = np.abs(v0).max()
    assert np.abs(v1 - v0).max() <= 1e-12 * scale
    assert not same(v0, v1)  # the variant really ran (fused rounding differs somewhere)
    assert np.abs(b1 - b0).max() <= 1e-12 * max(np.abs(b0).max(), 1.0)
    cfg = S.LevelConfig(degrees=[2, 1, 0], coarse="gmres-ilu", smoother="bjacobi",
                        outer_rtol=1e-8, restart=30)
    x0, h0, r0 = S.LevelHierarchy(A0, lay, cfg).solve(b0)
    x1, h1, r1 = S.LevelHierarchy(A1, lay1, cfg).solve(b1)
    assert r0.converged and r1.converged
    assert r1.outer_its == r0.outer_its and r1.coarse_its == r0.coarse_its  # tolerance: exact counts
    assert np.all(np.abs(h1 - h0) <= 1e-9 * np.abs(h0))  # tolerance 1e-9 relative
    assert np.abs(x1 - x0).max() <= 1e-9 * np.abs(x0).max()  # tolerance 1e-9 relative


@pytest.mark.parametrize("knobs", [
    {},                                   # default: dense-product face-block folds (PSCU_FLOW_BFAST=1)
    {"PSCU_FLOW_BFAST": "0"},             # general lane-0 / lane-parallel folds
    {"PSCU_FLOW_BSHFL": "1"},             # warp-replicated shuffle chain (backward)
    {"PSCU_FLOW_LEAD": "1"},              # lead-source wait before polling all
    {"PSCU_LEVEL_CHAIN_ROWS": "16"},      # element chains: mid-size dataflow kernel
    {"PSCU_LEVEL_CHAIN_ROWS": "16", "PSCU_FLOW_BSHFL": "1"},
    {"PSCU_LEVEL_PAD": "0"},              # unpadded rows: the dense / shuffle folds switch off
], ids=lambda k: "+".join(f"{a[5:]}={b}" for a, b in k.items()) or "default")
def test_dataflow_sweep_variants_bitwise_3d(M, knobs):
    _flow_variant_case(knobs, 5)


def test_dataflow_sweeps_bitwise_3d_8cubed(M):
    """The default folds on 8^3 (216 interior elements: mostly the uniform
    three-block face-block tasks the fixed straight-line paths serve)."""
    _flow_variant_case({}, 8)


def _flow_variant_case(knobs, n):
    """The barrier-free dataflow sweeps of the 3D coarse level (the path the
    benchmarked configs 3 / 5 run; small meshes would take the push walker,
    so the level plans are forced) under every fold variant: coarse ILU(0)
    V-cycle and the whole solve bit for bit against the oracle. A fresh
    process per variant (plan-time knobs)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import oracle_ref as O
from paper_2009_13840_b200 import host, solver as S
m = host.Mesh3(MESH_N, jitter=0.15, seed=1)
L = host.HpLocal3(2)
mats, rhs = L.local_blocks(m, 0, m.n_elements, data="random", seed=2)
brp, bcols = m.block_pattern()
rp, cols = O.bsr_to_csr_pattern(brp, bcols, L.face_block)
lay = O.po_layout(1, 2, 2, m.n_faces, m.n_elements, dim=3)
a, b = O.port_condense_assemble(mats, rhs, L.n_local, L.elim, L.kept_global(m.element_faces()), lay, rp, cols)
A, bd, lay_d, info = host.assemble_stokes3(m, 2, data="random", seed=2)
ref = O.PortHierarchy(a, lay, [2, 1, 0], smoother_iters=2, smoother=1)
cfg = S.LevelConfig(degrees=[2, 1, 0], coarse="gmres-ilu", smoother="bjacobi", outer_rtol=1e-8, restart=30)
h = S.LevelHierarchy(A, lay_d, cfg)
d = np.random.default_rng(4).standard_normal(a.n)
assert h.vcycle(0, d).tobytes() == ref.vcycle(0, d).tobytes()
r = ref.solve(b, rtol=1e-8, maxit=200, restart=30)
x, hist, rep = h.solve(bd)
assert rep.converged and rep.outer_its == r["its"] and rep.coarse_its == r["coarse_its"]
assert hist.tobytes() == r["hist"].tobytes() and x.tobytes() == r["x"].tobytes()
print("flow variants ok", rep.outer_its, rep.coarse_its)
'''
    env = dict(os.environ, PSCU_WALK_MODE="levels", PSCU_LEVEL_PERSIST_MIN_ROWS="0",
               PSCU_LEVEL_PERSIST="0", PSCU_LEVEL_FLOW="1", PSCU_DEBUG="1", **knobs)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code.replace("MESH_N", str(n))], cwd=root, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "flow variants ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    assert "cluster=1 level" in r.stderr, r.stderr[-2000:]  # the task-level (dataflow) plan was taken
