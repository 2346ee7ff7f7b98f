"""CPU tests of the 3D DG (BR2) producer — BASELINE.json config 4 — and its
oracle (host/pstokes_host3d.cpp DG section; oracle/pstokes_oracle.c
po_dg_pattern / po_dg_assemble restating assemble.hpp:177-346 with three
velocity components). The reference is 2D only; the 3D scheme is pinned by
(a) the structural pattern size SURVEY.md §8 G quotes for config 4, (b) the
DG block rows equal, bit for bit, to the oracle's reference-order scatter of
the same local terms, (c) manufactured-solution convergence, (d) the oracle
multilevel solve converging."""
import numpy as np
import pytest

import oracle_ref as O

pytestmark = pytest.mark.skipif(not O.port_available(), reason="oracle restatement not built")


@pytest.fixture(scope="module")
def host():
    from paper_2009_13840_b200 import build, host
    build.build_host()
    return host


def test_config4_pattern_size(host):
    # C4 DG k=3 at 32^3: 2,621,440 dofs / 892,928,000 structural nnz
    m = host.Mesh3(32, jitter=0.0, seed=3)
    D = host.DgLocal3(3)
    rp, cols = D.block_pattern(m)
    assert m.n_elements * D.elem_block == 2_621_440
    assert len(cols) * 10 * D.ne ** 2 == 892_928_000
    assert np.all(np.diff(rp) >= 4) and np.all(np.diff(rp) <= 7)


@pytest.mark.parametrize("n,k,jitter,data", [(2, 1, 0.0, "random"), (3, 2, 0.0, "random"),
                                             (2, 3, 0.0, "random"), (3, 2, 0.15, "manufactured")])
def test_dg_rows_equal_reference_order_scatter(host, n, k, jitter, data):
    m = host.Mesh3(n, jitter=jitter, seed=3)
    D = host.DgLocal3(k)
    lay = O.po_layout(2, 0, k, m.n_faces, m.n_elements, dim=3)
    vol, vr, fm, fr = D.local_terms(m, data=data, seed=3)
    a, b = O.port_dg_assemble(lay, m.faces(), vol, vr, fm, fr)
    brp, bc = D.block_pattern(m)
    assert a.nnz == len(bc) * 10 * D.ne ** 2
    dv, dr = D.rows(m, brp, bc, 0, m.n_elements, data=data, seed=3)
    cv = O.dgb_to_csr_values(a.row_ptr, brp, bc, dv, D.ne)
    assert cv.tobytes() == a.vals.tobytes()
    assert dr.tobytes() == b.tobytes()
    # split ranges give the same rows
    h = m.n_elements // 2
    d1, r1 = D.rows(m, brp, bc, 0, h, data=data, seed=3)
    d2, r2 = D.rows(m, brp, bc, h, m.n_elements, data=data, seed=3)
    assert np.concatenate([d1, d2]).tobytes() == dv.tobytes()
    assert np.concatenate([r1, r2]).tobytes() == dr.tobytes()


def test_velocity_block_symmetric(host):
    m = host.Mesh3(2, jitter=0.1, seed=3)
    D = host.DgLocal3(2)
    lay = O.po_layout(2, 0, 2, m.n_faces, m.n_elements, dim=3)
    a, _ = O.port_dg_assemble(lay, m.faces(), *D.local_terms(m, data="random", seed=3))
    A = a.to_dense()
    iv = np.array([r for r in range(a.n) if r % D.elem_block < 3 * D.ne])
    S = A[np.ix_(iv, iv)]
    assert np.abs(S - S.T).max() <= 1e-12 * np.abs(S).max()


@pytest.mark.parametrize("k,min_rate", [(1, 1.7), (2, 2.6)])
def test_manufactured_convergence(host, k, min_rate):
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    errs = []
    for n in (2, 4):
        m = host.Mesh3(n, jitter=0.0, seed=3)
        D = host.DgLocal3(k)
        lay = O.po_layout(2, 0, k, m.n_faces, m.n_elements, dim=3)
        a, b = O.port_dg_assemble(lay, m.faces(), *D.local_terms(m, data="manufactured"))
        A = sp.csr_matrix((a.vals, a.cols, a.row_ptr), shape=(a.n, a.n)).tocsc()
        errs.append(D.l2_errors(m, sla.spsolve(A, b)))
    rate_u = np.log2(errs[0][0] / errs[1][0])
    rate_p = np.log2(errs[0][1] / errs[1][1])
    assert rate_u > min_rate and rate_p > min_rate - 0.5, (errs, rate_u, rate_p)


def test_oracle_multilevel_solve_converges(host):
    m = host.Mesh3(3, jitter=0.0, seed=3)
    D = host.DgLocal3(3)
    lay = O.po_layout(2, 0, 3, m.n_faces, m.n_elements, dim=3)
    a, b = O.port_dg_assemble(lay, m.faces(), *D.local_terms(m, data="random", seed=3))
    r = O.PortHierarchy(a, lay, [3, 2, 1], smoother_iters=2, smoother=1).solve(
        b, rtol=1e-8, maxit=1000, restart=30)
    assert r["converged"] and r["its"] < 300
    res = b - a.to_dense() @ r["x"]
    assert np.linalg.norm(res) <= 1e-7 * np.linalg.norm(b)


def test_dg_layout_rules():
    with pytest.raises(ValueError):
        O.po_layout(2, 0, 0, 0, 8, dim=3)  # DG coarsest degree >= 1 (plevels.hpp:137-139)
    with pytest.raises(ValueError):
        O.po_layout(2, 1, 2, 0, 8, dim=3)  # no condensation for DG
    lay = O.po_layout(2, 0, 3, 0, 8, dim=3)
    assert (lay.elem_vel, lay.elem_press, lay.face_vel) == (20, 20, 0)
