"""The product's host input producer (include/pstokes_host.h) against the
reference front end: mesh / face numbering, eliminated dofs, retained
global ids and the CSR pattern must match exactly, and so must the local
blocks and loads, bit for bit: the producer evaluates every expression of
basis.hpp / hho_local.hpp in the order the reference's Eigen subset does
(left-to-right products, sums from 0, the fixed-shape reproducible dot)."""
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
        m = np.ascontiguousarray(mats[e].T)
        assert m.tobytes() == np.ascontiguousarray(m_ref).tobytes()
        assert np.ascontiguousarray(rhs[e]).tobytes() == np.ascontiguousarray(r_ref).tobytes()
        if loc.n_elim:
            assert np.array_equal(kept[e], ref.condensation(e)["kept_global"])


def test_benchmark_operator_digest_matches_reference_fixture(H):
    """Config 2a recipe at 64^2 through the product's host producer and the
    oracle's element-order condensation: the assembled operator and load
    hash to the reference solve's fixture (tests/golden/c2_vcond_64.json)."""
    import hashlib
    import json
    import os

    fx = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c2_vcond_64.json")))
    mesh = H.Mesh.unit_square(64, tri=True, jitter=0.2, seed=0, neumann="top")
    loc = H.LocalSystem(mesh, "hho-dp", "v-cond", 3, data="sincos")
    lay = O.po_layout(0, 1, 3, loc.n_faces, loc.nelem)
    a, b = O.port_condense_assemble(loc.mats(), loc.rhs(), loc.n_local, loc.elim(),
                                    loc.kept_global().reshape(loc.nelem, loc.n_keep), lay,
                                    loc.row_ptr(), loc.cols())

    def digest(*arrays):
        h = hashlib.sha256()
        for x in arrays:
            h.update(np.ascontiguousarray(x).tobytes())
        return h.hexdigest()

    assert digest(a.row_ptr, a.cols, a.vals) == fx["operator_sha256"]
    assert digest(b) == fx["rhs_sha256"]
