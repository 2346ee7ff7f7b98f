"""Oracle self-checks (CPU): pin the reference build against its own golden
values (proj/test_output.txt) and prove the plain-C restatement is
bit-identical to the reference on the solver path."""
import os

import numpy as np
import pytest

import oracle_ref as O

pytestmark = pytest.mark.skipif(not (O.ref_available() and O.port_available()),
                                reason="oracle libraries not built")

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def same(a, b):
    """Bitwise equality up to the sign of exact zeros (IEEE ==, no NaN)."""
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))


def test_acceptance_log_golden_iterations():
    """The acceptance run committed in tests/golden reproduces the
    reference's recorded iteration counts and dimensions
    (proj/test_output.txt:30,36-39)."""
    log = open(os.path.join(GOLDEN, "acceptance_eigen_subset.log")).read()
    assert "hho-dp/uncond=755712 hho-dp/vp-cond=280576 hho-dp/v-cond=428032 " \
           "hho-hp/vp-cond=396288 dg/uncond=491520" in log
    assert "(ITs = 6 7 7 7 7 7 )" in log
    assert "(ITs 7 -> 11)" in log
    assert "v-cond ITs = 16, v&p-cond ITs = 120* (cap 120)" in log
    assert "(rel diff 0 / 0)" in log
    assert "all criteria passed" in log


@pytest.mark.parametrize("n,its", [(2, 6), (4, 7), (8, 7)])
def test_reference_fgmres_iterations_golden(n, its):
    """Criterion 8 (acceptance.cpp:196-210): dp v-cond k=3 trapz, levels
    3/2/1, LU coarse, rtol 1e-13 -> ITs 6 7 7 ... (test_output.txt:37)."""
    s = O.RefSystem(family="trapz", n=n, k=3)
    r = s.solve_system([3, 2, 1], coarse="lu", rtol=1e-13)
    assert r["converged"] and r["its"] == its


def test_fgmres_hist_restatement_matches_solve_system():
    s = O.RefSystem(family="trapz", n=4, k=3)
    a = s.solve_system([3, 2, 1], coarse="lu", rtol=1e-13)
    b = s.solve([3, 2, 1], coarse="lu", rtol=1e-13)
    assert a["its"] == b["its"] and same(a["x"], b["x"]) and a["rel"] == b["rel"]


def test_layout_dims_golden():
    """Criterion 1 (acceptance.cpp:48-68) through the C restatement."""
    s = O.RefSystem(family="trapz", n=8, k=3)
    lay = s.layout
    for scheme, strat, want in [(0, 0, 755712), (0, 2, 280576), (0, 1, 428032), (1, 2, 396288),
                                (2, 0, 491520)]:
        # 16384-element trapz mesh: 128^2 quads, 33024 faces
        pl = O.po_layout(scheme, strat, 3, 2 * 128 * 129, 128 * 128)
        assert O.port_lib().po_layout_dim(pl) == want
    assert lay.n_elements == 64


CASES = [
    dict(family="trapz", n=3, scheme="hho-dp", strategy="v-cond", k=3, degrees=[3, 2, 1, 0]),
    dict(family="trapz", n=3, scheme="hho-dp", strategy="vp-cond", k=2, degrees=[2, 1, 0]),
    dict(family="tri", n=3, scheme="hho-hp", strategy="vp-cond", k=2, degrees=[2, 1, 0]),
    dict(family="trapz", n=2, scheme="dg", strategy="uncond", k=2, degrees=[2, 1]),
]


def _sys(c):
    return O.RefSystem(family=c["family"], n=c["n"], scheme=c["scheme"], strategy=c["strategy"],
                       k=c["k"])


def _port_layout(s):
    L = s.layout
    return O.po_layout(L.scheme, L.strategy, L.k, L.n_faces, L.n_elements)


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"{c['scheme']}-{c['strategy']}-k{c['k']}")
def test_port_spmv_ilu_bitwise(c):
    s = _sys(c)
    a = s.csr()
    rng = np.random.default_rng(1)
    x = rng.standard_normal(a.n)
    ra = O.RefCsr(a)
    y_ref = ra.multiply(x)
    y = np.zeros(a.n)
    pc = O.po_csr(a)
    O.port_lib().po_csr_multiply(pc, x, y)
    assert same(y, y_ref)
    ilu = O.RefIlu(ra)
    lu = np.zeros(a.nnz)
    diag = np.zeros(a.n, np.int64)
    assert O.port_lib().po_ilu0_factor(pc, lu, diag) == 0
    assert same(lu, ilu.factors())
    z = np.zeros(a.n)
    O.port_lib().po_ilu0_apply(pc, lu, diag, x, z)
    assert same(z, ilu.apply(x))


@pytest.mark.parametrize("c", CASES, ids=lambda c: f"{c['scheme']}-{c['strategy']}-k{c['k']}")
def test_port_hierarchy_vcycle_bitwise(c):
    s = _sys(c)
    a = s.csr()
    h_ref = O.RefHierarchy(s, c["degrees"], coarse="gmres-ilu")
    h = O.PortHierarchy(a, _port_layout(s), c["degrees"])
    for l in range(len(c["degrees"])):
        ra, pa = h_ref.level_csr(l), h.level_csr(l)
        assert same(ra.row_ptr, pa.row_ptr) and same(ra.cols, pa.cols) and same(ra.vals, pa.vals)
        assert same(h_ref.level_ilu(l), h.level_ilu(l))
    d = np.random.default_rng(3).standard_normal(a.n)
    assert same(h_ref.vcycle(0, d), h.vcycle(0, d))


@pytest.mark.parametrize("c", CASES[:3], ids=lambda c: f"{c['scheme']}-{c['strategy']}-k{c['k']}")
def test_port_solve_bitwise(c):
    s = _sys(c)
    r = s.solve(c["degrees"], coarse="gmres-ilu", rtol=1e-10)
    p = O.PortHierarchy(s.csr(), _port_layout(s), c["degrees"]).solve(s.rhs(), rtol=1e-10)
    assert r["its"] == p["its"] and r["coarse_its"] == p["coarse_its"]
    assert same(r["hist"], p["hist"]) and same(r["x"], p["x"])


def test_port_restart_consistent():
    """FGMRES(m) restart (BASELINE.json) is identical in the driver restatement
    and the C port."""
    s = O.RefSystem(family="trapz", n=3, scheme="hho-dp", strategy="vp-cond", k=2)
    r = s.solve([2, 1, 0], coarse="gmres-ilu", rtol=1e-12, restart=3)
    p = O.PortHierarchy(s.csr(), _port_layout(s), [2, 1, 0]).solve(s.rhs(), rtol=1e-12, restart=3)
    assert r["its"] == p["its"] and same(r["hist"], p["hist"]) and same(r["x"], p["x"])
    assert r["converged"]


def test_port_condense_bitwise():
    s = O.RefSystem(family="trapz", n=2, scheme="hho-dp", strategy="v-cond", k=2)
    for e in range(s.layout.n_elements):
        mat, rhs, elim = s.local_blocks(e, data="exp")
        ref = s.condensation(e)
        n = mat.shape[0]
        ne = len(elim)
        nk = n - ne
        schur = np.zeros(nk * nk)
        rr = np.zeros(nk)
        coup = np.zeros(ne * nk)
        er = np.zeros(ne)
        rc = O.port_lib().po_condense(n, np.asfortranarray(mat).ravel(order="F"), rhs, ne,
                                      np.ascontiguousarray(elim, np.int32), schur, rr, coup, er)
        assert rc == 0
        assert same(schur.reshape(nk, nk, order="F"), ref["schur"])
        assert same(rr, ref["reduced_rhs"])
        assert same(coup.reshape(ne, nk, order="F"), ref["elim_coupling"])
        assert same(er, ref["elim_rhs"])
