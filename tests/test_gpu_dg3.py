"""GPU parity of the 3D DG path (BASELINE.json config 4: BR2 DG, k = 3,
levels 3 -> 2 -> 1, V(2,2) block-Jacobi, ILU-GMRES coarse) against the
oracle restatement on identical host-built local terms: DG block storage
(csrc/dgb.cu) SpMV and CSR expansion, p-level inheritance of the panels,
block-Jacobi over 80 x 80 element blocks, V-cycles and full FGMRES solves,
the streamed assembly and the one-call drop-in. Bar: bitwise (IEEE ==)."""
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


def _system(host, n, k, jitter=0.0, data="random", seed=3):
    m = host.Mesh3(n, jitter=jitter, seed=3)
    D = host.DgLocal3(k)
    lay = O.po_layout(2, 0, k, m.n_faces, m.n_elements, dim=3)
    a, b = O.port_dg_assemble(lay, m.faces(), *D.local_terms(m, data=data, seed=seed))
    brp, bc = D.block_pattern(m)
    dv, dr = D.rows(m, brp, bc, 0, m.n_elements, data=data, seed=seed)
    return m, D, lay, a, b, brp, bc, dv, dr


@pytest.mark.parametrize("n,k", [(2, 1), (3, 2), (3, 3)])
def test_dgb_spmv_and_download_bitwise(M, n, k):
    host, S = M
    m, D, lay, a, b, brp, bc, dv, dr = _system(host, n, k)
    A = S.dgb_matrix(brp, bc, dv, D.ne)
    assert A.dg_modes == D.ne and A.n == a.n and A.nnz == a.nnz
    rp, cl, vl = A.download()
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(cl, a.cols) and same(vl, a.vals)
    rng = np.random.default_rng(n * 10 + k)
    for _ in range(3):
        x = rng.standard_normal(a.n)
        y = np.zeros(a.n)
        O.port_lib().po_csr_multiply(O.po_csr(a), x, y)
        assert same(A.multiply(x), y)


def test_dgb_inheritance_bitwise(M):
    host, S = M
    m, D, lay, a, b, brp, bc, dv, dr = _system(host, 3, 3)
    A = S.dgb_matrix(brp, bc, dv, D.ne)
    fine, Af, af = lay, A, a
    for kc in (2, 1):
        lc = S.make_layout3(kc, m.n_faces, m.n_elements, scheme="dg", strategy="uncond")
        lf = S.make_layout3(fine.k, m.n_faces, m.n_elements, scheme="dg", strategy="uncond")
        Ac = S.inherit_matrix(Af, lf, lc)
        assert Ac.dg_modes == (kc + 1) * (kc + 2) * (kc + 3) // 6
        pc = O.po_layout(2, 0, kc, m.n_faces, m.n_elements, dim=3)
        c2f = np.zeros(O.port_lib().po_layout_dim(pc), np.int64)
        O.port_lib().po_coarse_to_fine_map(fine, pc, c2f)
        assert same(S.coarse_to_fine_map(lf, lc), c2f)
        lib = O.port_lib()
        nc = len(c2f)
        nnz = lib.po_inherit(O.po_csr(af), af.n, c2f, nc, None, None, None)
        rp, cl, vl = np.zeros(nc + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
        lib.po_inherit(O.po_csr(af), af.n, c2f, nc, rp.ctypes.data, cl.ctypes.data, vl.ctypes.data)
        drp, dcl, dvl = Ac.download()
        assert np.array_equal(drp, rp) and np.array_equal(dcl, cl) and same(dvl, vl)
        fine, Af, af = pc, Ac, O.Csr(rp, cl, vl)


def test_block_jacobi_80_bitwise(M):
    host, S = M
    m, D, lay, a, b, brp, bc, dv, dr = _system(host, 3, 3)
    A = S.dgb_matrix(brp, bc, dv, D.ne)
    ld = S.make_layout3(3, m.n_faces, m.n_elements, scheme="dg", strategy="uncond")
    bj = S.BlockJacobi(A, ld)
    pbj = O.PortBlockJacobi(a, lay)
    x = np.random.default_rng(5).standard_normal(a.n)
    assert same(bj.apply(x), pbj.apply(x))


@pytest.mark.parametrize("n,k,degrees", [(3, 3, [3, 2, 1]), (4, 3, [3, 2, 1]), (3, 2, [2, 1])])
def test_dg_solve_bitwise(M, n, k, degrees):
    host, S = M
    m, D, lay, a, b, brp, bc, dv, dr = _system(host, n, k)
    A = S.dgb_matrix(brp, bc, dv, D.ne)
    ld = S.make_layout3(k, m.n_faces, m.n_elements, scheme="dg", strategy="uncond")
    cfg = S.LevelConfig(degrees=degrees, smoother="bjacobi", smoother_iters=2, coarse="gmres-ilu",
                        outer_rtol=1e-8, restart=30)
    H = S.LevelHierarchy(A, ld, cfg)
    P = O.PortHierarchy(a, lay, degrees, smoother_iters=2, smoother=1)
    d = np.random.default_rng(1).standard_normal(a.n)
    assert same(H.vcycle(0, d), P.vcycle(0, d))
    x, hist, rep = H.solve(dr)
    ref = P.solve(b, rtol=1e-8, maxit=1000, restart=30)
    assert rep.converged and rep.outer_its == ref["its"]
    assert same(hist, ref["hist"]) and same(x, ref["x"])


def test_streamed_assembly_and_dropin(M):
    host, S = M
    m, D, lay, a, b, brp, bc, dv, dr = _system(host, 4, 3)
    A, rhs, ld, info = host.assemble_dg3(m, 3, data="random", seed=3, batch=5)
    assert same(rhs, dr)
    _, _, vl = A.download()
    assert same(vl, a.vals)
    cfg = S.LevelConfig(degrees=[3, 2, 1], smoother="bjacobi", smoother_iters=2,
                        coarse="gmres-ilu", outer_rtol=1e-8, restart=30)
    x1, h1, r1 = S.LevelHierarchy(A, ld, cfg).solve(rhs)
    x2, h2, r2 = S.solve_system_dgb(brp, bc, dv, D.ne, dr, ld, cfg)
    assert r1.outer_its == r2.outer_its and same(h1, h2) and same(x1, x2)
