"""The product's host input producer (include/pstokes_host.h) against the
reference front end: mesh / face numbering, eliminated dofs, retained
global ids and the CSR pattern must match exactly; local blocks and loads
to 1e-11 relative (independent arithmetic order)."""
import numpy as np
import pytest

import oracle_ref as O
from paper_2009_13840_b200 import build

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="reference oracle not built")


@pytest.fixture(scope="module")
def H():
    build.build_host()
    from paper_2009_13840_b200 import host
    return host


CASES = [
    # (mesh kind, args, scheme, strategy, k, data)
    ("unit-quad", dict(n=4, side="top"), "hho-dp", "v-cond", 1, "sincos"),
    ("unit-tri", dict(n=4, jitter=0.2, seed=0, side="top"), "hho-dp", "v-cond", 3, "sincos"),
    ("unit-tri", dict(n=3, jitter=0.2, seed=0, side="top"), "hho-dp", "vp-cond", 3, "sincos"),
    ("family-trapz", dict(n=3, side="right"), "hho-dp", "v-cond", 2, "exp"),
    ("family-tri", dict(n=2, side="right"), "hho-hp", "vp-cond", 2, "exp"),
    ("family-quad", dict(n=2, side="right"), "hho-dp", "uncond", 1, "exp"),
    ("family-trapz", dict(n=2, side="right"), "hho-hp", "uncond", 1, "exp"),
]
IDS = [f"{c[0]}-{c[2]}-{c[3]}-k{c[4]}" for c in CASES]


def make(H, c):
    kind, a, scheme, strat, k, data = c
    if kind.startswith("family"):
        fam = kind.split("-")[1]
        ref = O.RefSystem(family=fam, n=a["n"], side=a["side"], scheme=scheme, strategy=strat,
                          k=k, data=data)
        mesh = H.Mesh.family(fam, a["n"], neumann=a["side"])
    else:
        ref = O.RefSystem(mesh=kind, n=a["n"], seed=a.get("seed", 0), jitter=a.get("jitter", 0.0),
                          side=a["side"], scheme=scheme, strategy=strat, k=k, data=data)
        mesh = H.Mesh.unit_square(a["n"], tri=kind == "unit-tri", jitter=a.get("jitter", 0.0),
                                  seed=a.get("seed", 0), neumann=a["side"])
    loc = H.LocalSystem(mesh, scheme, strat, k, data=data, nthreads=2)
    return ref, mesh, loc


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_mesh_and_numbering_exact(H, c):
    ref, mesh, loc = make(H, c)
    rm = ref.mesh()
    assert np.array_equal(mesh.faces(), rm["faces"])
    assert np.array_equal(mesh.vertices(), rm["xy"])
    assert loc.dim == ref.n
    L = ref.layout
    assert (loc.face_vel, loc.face_press, loc.elem_vel, loc.elem_press) == \
        (L.face_vel, L.face_press, L.elem_vel, L.elem_press)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_pattern_exact(H, c):
    ref, mesh, loc = make(H, c)
    a = ref.csr()
    assert np.array_equal(loc.row_ptr(), a.row_ptr)
    assert np.array_equal(loc.cols(), a.cols)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_local_blocks(H, c):
    ref, mesh, loc = make(H, c)
    n = loc.n_local
    mats = loc.mats().reshape(loc.nelem, n, n)  # [e, j, i] (column-major blocks)
    rhs = loc.rhs().reshape(loc.nelem, n)
    kept = loc.kept_global().reshape(loc.nelem, loc.n_keep)
    for e in range(loc.nelem):
        m_ref, r_ref, el_ref = ref.local_blocks(e, data=c[5])
        assert np.array_equal(loc.elim(), el_ref)
        m = mats[e].T
        scale = np.max(np.abs(m_ref))
        assert np.max(np.abs(m - m_ref)) <= 1e-11 * scale
        assert np.max(np.abs(rhs[e] - r_ref)) <= 1e-11 * max(np.max(np.abs(r_ref)), 1e-300) + 1e-14
        if loc.n_elim:
            assert np.array_equal(kept[e], ref.condensation(e)["kept_global"])
