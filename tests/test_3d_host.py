"""3D HHO-hp producer (host/pstokes_host3d.cpp, BASELINE.json configs 3 and
5) and the oracle's 3D path on the CPU: mesh topology and geometry, the
face-block pattern, local-block structure, and a manufactured-solution
solve through the C restatement (condensation, element-order assembly,
block-Jacobi-smoothed p-multigrid, ILU-GMRES coarse, FGMRES) whose face
errors converge under refinement. The reference has no 3D (mesh.hpp:21,
SPEC.md:8); these checks pin the 3D generalisation itself."""
import numpy as np
import pytest

import oracle_ref as O
from paper_2009_13840_b200 import build, host

pytestmark = pytest.mark.skipif(not O.port_available(), reason="oracle restatement not built")


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build_host()


def test_mesh_topology_and_geometry():
    for n, jit in [(1, 0.0), (3, 0.0), (4, 0.15)]:
        m = host.Mesh3(n, jitter=jit, seed=1)
        assert m.n_elements == n ** 3 and m.n_vertices == (n + 1) ** 3
        assert m.n_faces == 3 * n * n * (n + 1)
        f = m.faces()
        interior = f[:, 5] >= 0
        assert interior.sum() == 3 * n * n * (n - 1)
        assert np.all(f[interior, 6] == 0)
        # Neumann exactly on z = 1
        v = m.vertices()
        top = np.all(v[f[:, :4], 2] == 1.0, axis=1)
        assert np.all(f[top, 6] == 2) and np.all(f[~top & ~interior, 6] == 1)
        # first-seen numbering: face ids appear in increasing order over the element loop
        ef = m.element_faces().ravel()
        first = np.unique(ef, return_index=True)[1]
        assert np.all(np.diff(first) > 0)
        vol, clo = m.geometry()
        assert abs(vol.sum() - 1.0) < 1e-13 and clo.max() < 1e-15
        assert vol.min() > 0


def test_jitter_recipe_and_determinism():
    a, b = host.Mesh3(4, jitter=0.15, seed=1), host.Mesh3(4, jitter=0.15, seed=1)
    va, vb = a.vertices(), b.vertices()
    assert np.array_equal(va, vb)
    u = host.Mesh3(4).vertices()
    d = np.abs(va - u).max(axis=1)
    boundary = np.any((u == 0.0) | (u == 1.0), axis=1)
    assert np.all(d[boundary] == 0.0) and 0 < d[~boundary].max() <= 0.15 / 4


def test_block_pattern():
    m = host.Mesh3(3)
    rp, cols = m.block_pattern()
    f = m.faces()
    ef = m.element_faces()
    for face in range(m.n_faces):
        want = set(ef[f[face, 4]])
        if f[face, 5] >= 0:
            want |= set(ef[f[face, 5]])
        got = cols[rp[face]:rp[face + 1]]
        assert list(got) == sorted(want)
    # 11 block columns on interior faces, 6 on boundary faces
    assert set(np.diff(rp)) == {6, 11}


@pytest.mark.parametrize("k", [0, 1, 2])
def test_local_structure(k):
    L = host.HpLocal3(k)
    nf = (k + 1) * (k + 2) // 2
    ne = (k + 2) * (k + 3) * (k + 4) // 6
    npr = (k + 1) * (k + 2) * (k + 3) // 6
    assert L.face_block == 4 * nf and L.n_keep == 6 * 4 * nf
    assert L.n_elim == 3 * ne + npr and L.n_local == L.n_keep + L.n_elim
    if k == 2:
        assert (L.n_local, L.n_elim, L.n_keep, L.face_block) == (214, 70, 144, 24)
    m = host.Mesh3(2, jitter=0.1, seed=3)
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data="random", seed=2)
    n = L.n_local
    A = mats[: n * n].reshape(n, n, order="F")
    # the eliminated block is invertible and the viscous block symmetric
    E = A[np.ix_(L.elim, L.elim)]
    assert np.linalg.cond(E) < 1e12
    nv = 3 * (L.ne + 6 * nf)
    assert np.allclose(A[:nv, :nv], A[:nv, :nv].T, rtol=0, atol=1e-9 * np.abs(A).max())
    # kept global ids cover every face dof exactly once per incident element
    kept = L.kept_global(m.element_faces())
    cnt = np.bincount(kept.ravel(), minlength=m.n_faces * L.face_block)
    f = m.faces()
    per_face = np.where(f[:, 5] >= 0, 2, 1)
    assert np.array_equal(cnt.reshape(m.n_faces, -1), np.repeat(per_face[:, None], L.face_block, 1))
    # element-major random loads: a range build equals the full build
    m2, r2 = L.local_blocks(m, 3, 6, data="random", seed=2)
    assert np.array_equal(m2, mats[3 * n * n: 6 * n * n]) and np.array_equal(r2, rhs[3 * n: 6 * n])


def _solve3(n, jitter, k=2):
    m = host.Mesh3(n, jitter=jitter, seed=1)
    L = host.HpLocal3(k)
    mats, rhs = L.local_blocks(m, 0, m.n_elements, data="manufactured")
    brp, bcols = m.block_pattern()
    rp, cols = O.bsr_to_csr_pattern(brp, bcols, L.face_block)
    lay = O.po_layout(1, 2, k, m.n_faces, m.n_elements, dim=3)
    a, b = O.port_condense_assemble(mats, rhs, L.n_local, L.elim, L.kept_global(m.element_faces()),
                                    lay, rp, cols)
    h = O.PortHierarchy(a, lay, list(range(k, -1, -1)), smoother_iters=2, smoother=1)
    r = h.solve(b, rtol=1e-10, maxit=200, restart=30)
    x = r["x"].reshape(m.n_faces, -1)
    p = m.face_projection(k).reshape(m.n_faces, -1)
    nfv = 3 * L.face_vel
    err = np.sqrt(np.sum((x[:, :nfv] - p[:, :nfv]) ** 2) / m.n_faces)
    return r, err


def test_manufactured_solution_converges():
    """u = (sin pi y sin pi z, sin pi x sin pi z, sin pi x sin pi y),
    p = sin 2pi x sin 2pi y sin 2pi z on jittered hexahedra (non-planar
    faces): FGMRES converges and the face-velocity error against the face
    L2 projections drops by > 2^4 per refinement (k = 2)."""
    r2, e2 = _solve3(2, 0.15)
    r4, e4 = _solve3(4, 0.15)
    assert r2["converged"] and r4["converged"]
    assert e2 / e4 > 16.0, (e2, e4)
