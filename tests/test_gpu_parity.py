"""GPU parity: the sm_100a path (through the C ABI) against the oracles on
identical inputs. Bar: bit-exact (IEEE ==, i.e. up to the sign of exact
zeros) for SpMV, ILU(0), transfers, inheritance, GMRES/FGMRES, V-cycle,
condensation and full solves with the reproducible dot shared with the
oracle; iteration counts equal everywhere; residual histories and
solutions within 1e-9 relative (north_star) where a different coarse LU
is used (dense device LU vs the reference's sparse LU)."""
import numpy as np
import pytest

import oracle_ref as O
import synthetic

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (O.ref_available() and O.port_available()),
                                 reason="oracle libraries not built")]


@pytest.fixture(scope="module")
def S():
    from paper_2009_13840_b200 import solver
    return solver


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and bool(np.all(a == b))


def rel_close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(np.max(np.abs(b)), 1e-300)
    return a.shape == b.shape and float(np.max(np.abs(a - b))) <= tol * scale


CASES = [
    dict(family="trapz", n=4, scheme="hho-dp", strategy="v-cond", k=3, degrees=[3, 2, 1, 0]),
    dict(family="trapz", n=3, scheme="hho-dp", strategy="vp-cond", k=2, degrees=[2, 1, 0]),
    dict(family="tri", n=3, scheme="hho-hp", strategy="vp-cond", k=2, degrees=[2, 1, 0]),
    dict(family="graded-tri", n=4, scheme="hho-dp", strategy="v-cond", k=1, degrees=[1, 0]),
    dict(family="trapz", n=2, scheme="dg", strategy="uncond", k=2, degrees=[2, 1]),
]
IDS = [f"{c['family']}-{c['scheme']}-{c['strategy']}-k{c['k']}" for c in CASES]


def _sys(c, **kw):
    return O.RefSystem(family=c["family"], n=c["n"], scheme=c["scheme"], strategy=c["strategy"],
                       k=c["k"], **kw)


def _layout(S, s):
    L = s.layout
    return S.make_layout(L.scheme, L.strategy, L.k, L.n_faces, L.n_elements)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_spmv_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    x = np.random.default_rng(0).standard_normal(a.n)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    assert same(m.multiply(x), O.RefCsr(a).multiply(x))
    rp, cl, vl = m.download()
    assert same(rp, a.row_ptr) and same(cl, a.cols) and same(vl, a.vals)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_ilu0_factor_and_apply_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    assert same(ilu.factors(), ri.factors())
    x = np.random.default_rng(1).standard_normal(a.n)
    assert same(ilu.apply(x), ri.apply(x))


def test_ilu0_zero_pivot_raises(S):
    # [[0, 1], [1, 0]] has an explicit zero diagonal: ilu0.hpp:46-47 throws
    m = S.CsrMatrix(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([0.0, 1.0, 1.0, 0.0]))
    with pytest.raises(RuntimeError, match="zero pivot"):
        S.Ilu0(m)


def test_ilu0_missing_diagonal_raises(S):
    m = S.CsrMatrix(np.array([0, 1, 2]), np.array([1, 0]), np.array([1.0, 1.0]))
    with pytest.raises(RuntimeError, match="no diagonal"):
        S.Ilu0(m)


@pytest.mark.parametrize("side", ["right", "left"])
@pytest.mark.parametrize("c", CASES[:3], ids=IDS[:3])
def test_gmres_bitwise(S, c, side):
    s = _sys(c)
    a = s.csr()
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    rng = np.random.default_rng(2)
    b = rng.standard_normal(a.n)
    x0 = rng.standard_normal(a.n)
    for (maxit, rtol) in [(2, 0.0), (40, 1e-6)]:
        r = O.ref_gmres(ra, ri, b, x0, maxit, rtol, left=side == "left")
        g = S.gmres(m, ilu, b, x0, maxit, rtol, side=side)
        assert g.iterations == r["its"] and g.converged == r["converged"]
        assert g.rel_residual == r["rel"]
        assert same(g.x, r["x"])


def test_gmres_zero_x0_and_zero_rhs(S):
    s = _sys(CASES[0])
    a = s.csr()
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    b = np.random.default_rng(4).standard_normal(a.n)
    r = O.ref_gmres(ra, ri, b, np.zeros(a.n), 30, 1e-8)
    g = S.gmres(m, ilu, b, None, 30, 1e-8)
    assert g.iterations == r["its"] and same(g.x, r["x"])
    g0 = S.gmres(m, ilu, np.zeros(a.n), None, 5, 0.0)
    assert g0.converged and g0.iterations == 0 and not np.any(g0.x)


@pytest.mark.parametrize("c", CASES[:3], ids=IDS[:3])
def test_fgmres_fixed_preconditioner_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    b = np.random.default_rng(5).standard_normal(a.n)
    r = O.ref_fgmres(ra, ri, b, 60, 1e-10)
    g = S.fgmres(m, ilu, b, 60, 1e-10)
    assert g.iterations == r["its"] and g.converged == r["converged"]
    assert g.rel_residual == r["rel"] and same(g.x, r["x"])
    # unconverged runs are reported with iterations == cap (test_sparse_la.cpp:167-173)
    g3 = S.fgmres(m, None, b, 3, 1e-15)
    assert not g3.converged and g3.iterations == 3


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_layouts_transfers_inheritance_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    lf = _layout(S, s)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    for kc in c["degrees"][1:]:
        ref, c2f = s.inherit(c["k"], kc)
        lc = S.make_layout(s.layout.scheme, s.layout.strategy, kc, s.layout.n_faces,
                           s.layout.n_elements)
        assert S.layout_dim(lc) == s.layout_dim(kc)
        assert same(S.coarse_to_fine_map(lf, lc), c2f)
        inh = S.inherit_matrix(m, lf, lc)
        rp, cl, vl = inh.download()
        assert same(rp, ref.row_ptr) and same(cl, ref.cols) and same(vl, ref.vals)


def test_layout_validation(S):
    with pytest.raises(ValueError):
        S.make_layout("hho-hp", "v-cond", 2, 10, 4)
    with pytest.raises(ValueError):
        S.make_layout("dg", "uncond", 0, 10, 4)


@pytest.mark.parametrize("c", CASES, ids=IDS)
def test_hierarchy_and_vcycle_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    href = O.RefHierarchy(s, c["degrees"], coarse="gmres-ilu")
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    cfg = S.LevelConfig(degrees=c["degrees"], coarse="gmres-ilu")
    h = S.LevelHierarchy(m, _layout(S, s), cfg)
    for l in range(len(c["degrees"])):
        rp, cl, vl = h.level_matrix(l).download()
        ref = href.level_csr(l)
        assert same(vl, ref.vals) and same(cl, ref.cols)
        assert same(h.level_ilu(l).factors(), href.level_ilu(l))
    d = np.random.default_rng(6).standard_normal(a.n)
    href.reset()
    h.reset_counters()
    assert same(h.vcycle(0, d), href.vcycle(0, d))
    assert h.coarse_iterations() == href.coarse_its()
    # zero defect gives a zero correction; homogeneity (test_plevels.cpp:131-151)
    assert not np.any(h.vcycle(0, np.zeros(a.n)))
    c1, c3 = h.vcycle(0, d), h.vcycle(0, 3.0 * d)
    assert np.max(np.abs(c3 - 3 * c1)) <= 1e-12 * np.max(np.abs(c1)) * 3


def test_level_validation(S):
    s = _sys(CASES[0])
    a = s.csr()
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    for deg in ([3, 3], [4, 1], [3, 2, 2]):
        with pytest.raises(ValueError):
            S.LevelHierarchy(m, _layout(S, s), S.LevelConfig(degrees=deg))


@pytest.mark.parametrize("c", CASES[:4], ids=IDS[:4])
def test_full_solve_bitwise(S, c):
    """solve_system with the ILU-GMRES coarse solver: identical ITs, coarse
    ITs, residual history and solution."""
    s = _sys(c, data="exp")
    a = s.csr()
    r = s.solve(c["degrees"], coarse="gmres-ilu", rtol=1e-10)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    h = S.LevelHierarchy(m, _layout(S, s), S.LevelConfig(degrees=c["degrees"], coarse="gmres-ilu",
                                                         outer_rtol=1e-10))
    x, hist, rep = h.solve(s.rhs())
    assert rep.outer_its == r["its"] and rep.coarse_its == r["coarse_its"]
    assert rep.vcycles == r["vcycles"] and rep.converged == r["converged"]
    assert same(hist, r["hist"]) and same(x, r["x"])


def test_golden_iterations_lu_coarse(S):
    """Criterion 8 known answers (test_output.txt:37) with the reference's
    default coarse LU replaced by the device dense LU: ITs 6, 7, 7 on trapz
    n=2,4,8 at rtol 1e-13, levels 3/2/1; history within 1e-9 of the
    reference's."""
    for n, its in [(2, 6), (4, 7), (8, 7)]:
        s = O.RefSystem(family="trapz", n=n, k=3)
        r = s.solve([3, 2, 1], coarse="lu", rtol=1e-13)
        a = s.csr()
        m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
        h = S.LevelHierarchy(m, _layout(S, s), S.LevelConfig(degrees=[3, 2, 1], coarse="lu"))
        x, hist, rep = h.solve(s.rhs())
        assert rep.converged and rep.outer_its == its == r["its"]
        # 1e-9 relative wherever the estimate is above 1e-10 of ||b||; the
        # last entries sit at roundoff (rtol 1e-13) where the dense device LU
        # and the reference's sparse LU round differently: 1e-3 relative there
        ref_h = np.asarray(r["hist"])
        rel = np.abs(hist - ref_h) / np.abs(ref_h)
        big = ref_h >= 1e-10
        assert np.all(rel[big] <= 1e-9) and np.all(rel[~big] <= 1e-3), rel
        assert rel_close(x, r["x"], 1e-9)


def test_config1_unit_square(S):
    """BASELINE.json config 1 (16x16 quads, k=1, levels 1->0, sin/cos field,
    Neumann top): solve_system through the one-call C ABI entry."""
    s = O.RefSystem(mesh="unit-quad", n=16, side="top", k=1, data="sincos")
    a = s.csr()
    for coarse in ("lu", "gmres-ilu"):
        r = s.solve([1, 0], coarse=coarse, rtol=1e-8)
        cfg = S.LevelConfig(degrees=[1, 0], coarse=coarse, outer_rtol=1e-8)
        x, hist, rep = S.solve_system(a.row_ptr, a.cols, a.vals, s.rhs(), _layout(S, s), cfg)
        assert rep.converged and rep.outer_its == r["its"] == 5
        if coarse == "gmres-ilu":
            assert same(hist, r["hist"]) and same(x, r["x"])
            assert rep.coarse_its == r["coarse_its"]
        else:
            assert rel_close(x, r["x"], 1e-9)


def test_fgmres_restart(S):
    c = CASES[1]
    s = _sys(c)
    a = s.csr()
    r = s.solve(c["degrees"], coarse="gmres-ilu", rtol=1e-12, restart=3)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    h = S.LevelHierarchy(m, _layout(S, s), S.LevelConfig(degrees=c["degrees"], coarse="gmres-ilu",
                                                         outer_rtol=1e-12, restart=3))
    x, hist, rep = h.solve(s.rhs())
    assert rep.outer_its == r["its"] and same(hist, r["hist"]) and same(x, r["x"])


@pytest.mark.parametrize("scheme,strategy,k", [("hho-dp", "v-cond", 2), ("hho-dp", "vp-cond", 3),
                                               ("hho-hp", "vp-cond", 1)])
def test_condensation_bitwise(S, scheme, strategy, k):
    s = O.RefSystem(family="trapz", n=2, scheme=scheme, strategy=strategy, k=k)
    ne_el = s.layout.n_elements
    mats, rhss, refs = [], [], []
    elim0 = None
    for e in range(ne_el):
        mat, rhs, elim = s.local_blocks(e, data="exp")
        elim0 = elim if elim0 is None else elim0
        assert same(elim, elim0)
        mats.append(mat)
        rhss.append(rhs)
        refs.append(s.condensation(e))
    out = S.condense_elements(np.stack(mats), np.stack(rhss), elim0)
    for e in range(ne_el):
        assert same(out["schur"][e], refs[e]["schur"])
        assert same(out["reduced_rhs"][e], refs[e]["reduced_rhs"])
        assert same(out["elim_coupling"][e], refs[e]["elim_coupling"])
        assert same(out["elim_rhs"][e], refs[e]["elim_rhs"])


def _recover_ref(coup, erhs, kept_vals):
    """ElementCondensation::recover (condense.hpp:28-38) as the reference
    computes it: xe = elim_rhs - elim_coupling * kept, the product summed k
    ascending from 0.0 (include/eigen_subset GEMM), one rounding per op."""
    ne, nk = coup.shape
    out = np.zeros(ne)
    for i in range(ne):
        acc = 0.0
        for k in range(nk):
            acc = acc + float(coup[i, k]) * float(kept_vals[k])
        out[i] = float(erhs[i]) - acc
    return out


@pytest.mark.parametrize("family,scheme,strategy,k", [("trapz", "hho-dp", "v-cond", 3),
                                                      ("trapz", "hho-dp", "vp-cond", 2),
                                                      ("tri", "hho-hp", "vp-cond", 2),
                                                      ("trapz", "hho-hp", "vp-cond", 1)])
def test_recovery_bitwise(S, family, scheme, strategy, k):
    """pscu_recover_batch (recover_kernel) against the reference's recovery
    data and back-substitution, every element, a random global vector."""
    s = O.RefSystem(family=family, n=3, scheme=scheme, strategy=strategy, k=k)
    ne_el = s.layout.n_elements
    refs = [s.condensation(e) for e in range(ne_el)]
    _, _, elim = s.local_blocks(0, data="exp")
    x = np.random.default_rng(7).standard_normal(s.n)
    kept = np.stack([r["kept_global"] for r in refs])
    coup = np.stack([r["elim_coupling"] for r in refs])
    erhs = np.stack([r["elim_rhs"] for r in refs])
    got = S.recover_elements(elim, kept, coup, erhs, x)
    n = kept.shape[1] + len(elim)
    is_elim = np.zeros(n, bool)
    is_elim[elim] = True
    keep = np.nonzero(~is_elim)[0]
    for e in range(ne_el):
        want = np.zeros(n)
        want[keep] = x[kept[e]]
        want[elim] = _recover_ref(coup[e], erhs[e], x[kept[e]])
        assert same(got[e], want), e


def test_condensation_singular_block_raises(S):
    n = 4
    mats = np.stack([np.eye(n), np.eye(n)])
    mats[1, 0, 0] = 0.0  # eliminated dof 0 has a zero pivot on element 1
    with pytest.raises(RuntimeError, match="element 1"):
        S.condense_elements(mats, np.ones((2, n)), [0])


# Sweep-plan variants (walk.cu): the push walker over row chains (default on
# narrow sweeps), task-level launches (default on wide sweeps; warp- and
# thread-per-task kernels), the level walker and row (chain-free) plans.
# Every variant must reproduce Ilu0::apply bitwise.
PLAN_MODES = [("default", "16"), ("default", "3"), ("default", "1"), ("levels", "16"),
              ("levels", "1"), ("walker", "1"), ("push1", "16")]
PLAN_CASES = [dict(mesh="unit-tri", n=12, jitter=0.2, seed=0, side="top", scheme="hho-dp",
                   strategy="v-cond", k=3, data="sincos"),
              dict(mesh="unit-tri", n=16, jitter=0.2, seed=0, side="top", scheme="hho-dp",
                   strategy="v-cond", k=0, data="sincos"),
              dict(family="trapz", n=6, scheme="hho-dp", strategy="vp-cond", k=2)]


@pytest.mark.parametrize("mode,rows", PLAN_MODES, ids=[f"{m}-g{r}" for m, r in PLAN_MODES])
@pytest.mark.parametrize("ci", range(len(PLAN_CASES)))
def test_ilu0_plan_variants_bitwise(S, monkeypatch, mode, rows, ci):
    if mode != "default":
        monkeypatch.setenv("PSCU_WALK_MODE", mode)
    monkeypatch.setenv("PSCU_CHAIN_ROWS", rows)
    monkeypatch.setenv("PSCU_LEVEL_CHAIN_ROWS", rows)
    s = O.RefSystem(**PLAN_CASES[ci])
    a = s.csr()
    ri = O.RefIlu(O.RefCsr(a))
    ilu = S.Ilu0(S.CsrMatrix(a.row_ptr, a.cols, a.vals))
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert same(ilu.apply(x), ri.apply(x))


@pytest.mark.parametrize("ci", range(len(PLAN_CASES)))
def test_ilu0_single_cta_dataflow_walker_bitwise(S, monkeypatch, ci):
    """The single-CTA dataflow walker (walk.cu flow_kernel: chunks span task
    levels, rows wait on their own sources; PSCU_WALK_FLOW with a one-CTA
    cluster) reproduces Ilu0::apply bitwise."""
    monkeypatch.setenv("PSCU_WALK_CLUSTER", "1")
    monkeypatch.setenv("PSCU_WALK_FLOW", "1")
    s = O.RefSystem(**PLAN_CASES[ci])
    a = s.csr()
    ri = O.RefIlu(O.RefCsr(a))
    ilu = S.Ilu0(S.CsrMatrix(a.row_ptr, a.cols, a.vals))
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert ilu.apply(x).tobytes() == ri.apply(x).tobytes()


# Block-Jacobi over entity blocks (BASELINE.json's smoother; a labelled
# alternative to the reference's ILU(0), oracle: po_bj_* / po_hier_create_ex
# in oracle/pstokes_oracle.c). Apply, V-cycle and full solves bitwise.
BJ_CASES = [dict(family="tri", n=4, scheme="hho-hp", strategy="vp-cond", k=3, degrees=[3, 2, 1, 0]),
            dict(family="trapz", n=3, scheme="hho-hp", strategy="vp-cond", k=2, degrees=[2, 1, 0]),
            dict(family="trapz", n=2, scheme="dg", strategy="uncond", k=2, degrees=[2, 1])]
BJ_IDS = [f"{c['family']}-{c['scheme']}-k{c['k']}" for c in BJ_CASES]


def _po_layout(s):
    L = s.layout
    return O.po_layout(L.scheme, L.strategy, L.k, L.n_faces, L.n_elements)


@pytest.mark.parametrize("c", BJ_CASES, ids=BJ_IDS)
def test_bjacobi_apply_bitwise(S, c):
    s = _sys(c)
    a = s.csr()
    ref = O.PortBlockJacobi(a, _po_layout(s))
    bj = S.BlockJacobi(S.CsrMatrix(a.row_ptr, a.cols, a.vals), _layout(S, s))
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert same(bj.apply(x), ref.apply(x))


def test_bjacobi_singular_block_raises(S):
    # HHO-dp v-cond: the element mean-pressure block is singular (SURVEY.md
    # §0 finding 4); both sides refuse it
    s = _sys(CASES[1] | dict(strategy="v-cond"))
    a = s.csr()
    with pytest.raises(RuntimeError, match="singular"):
        O.PortBlockJacobi(a, _po_layout(s))
    with pytest.raises(RuntimeError, match="singular"):
        S.BlockJacobi(S.CsrMatrix(a.row_ptr, a.cols, a.vals), _layout(S, s))


@pytest.mark.parametrize("c", BJ_CASES, ids=BJ_IDS)
def test_bjacobi_vcycle_and_solve_bitwise(S, c):
    s = _sys(c, data="exp")
    a = s.csr()
    ref = O.PortHierarchy(a, _po_layout(s), c["degrees"], smoother=1)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    cfg = S.LevelConfig(degrees=c["degrees"], coarse="gmres-ilu", smoother="bjacobi",
                        outer_rtol=1e-10)
    h = S.LevelHierarchy(m, _layout(S, s), cfg)
    d = np.random.default_rng(3).standard_normal(a.n)
    assert same(h.vcycle(0, d), ref.vcycle(0, d))
    r = ref.solve(s.rhs(), rtol=1e-10)
    x, hist, rep = h.solve(s.rhs())
    assert rep.converged and r["converged"]
    assert rep.outer_its == r["its"] and rep.coarse_its == r["coarse_its"]
    assert same(hist, r["hist"]) and same(x, r["x"])


@pytest.mark.parametrize("tma,allg", [("0", "0"), ("0", "1"), ("1", "0")])
@pytest.mark.parametrize("side", ["right", "left"])
def test_gmres_mgs_variants_bitwise(S, monkeypatch, tma, allg, side):
    """The fused Arnoldi step: root-CTA and all-gather grid reductions, and
    the basis streamed through shared memory by TMA (arnoldi_tma_kernel;
    forced at small sizes)."""
    monkeypatch.setenv("PSCU_MGS_TMA_MIN_G", "1")
    monkeypatch.setenv("PSCU_MGS_TMA", tma)
    monkeypatch.setenv("PSCU_MGS_ALL", allg)
    s = O.RefSystem(**PLAN_CASES[0])
    a = s.csr()
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(a.n)
    x0 = rng.standard_normal(a.n)
    for (maxit, rtol) in [(3, 0.0), (60, 1e-9)]:
        r = O.ref_gmres(ra, ri, b, x0, maxit, rtol, left=side == "left")
        g = S.gmres(m, ilu, b, x0, maxit, rtol, side=side)
        assert g.iterations == r["its"] and g.converged == r["converged"]
        assert same(g.x, r["x"])


def test_gmres_wide_grid_reduction_bitwise(S):
    """A size where the fused Arnoldi step's grid reduction runs over 64 CTAs
    (warp 0 of every CTA gathers two CTA partials per lane): 128^2 tris, k=0."""
    s = O.RefSystem(mesh="unit-tri", n=128, jitter=0.2, seed=0, side="top", scheme="hho-dp",
                    strategy="v-cond", k=0, data="sincos")
    a = s.csr()
    assert a.n > 16 * 256 * 32
    ra = O.RefCsr(a)
    ri = O.RefIlu(ra)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    ilu = S.Ilu0(m)
    b = np.random.default_rng(7).standard_normal(a.n)
    x0 = np.zeros(a.n)
    r = O.ref_gmres(ra, ri, b, x0, 25, 0.0, left=False)
    g = S.gmres(m, ilu, b, x0, 25, 0.0, side="right")
    assert g.iterations == r["its"] and same(g.x, r["x"])


@pytest.mark.parametrize("thread_rows", ["0", "1"])
@pytest.mark.parametrize("ci", range(len(PLAN_CASES)))
def test_ilu0_factor_variants_bitwise(S, monkeypatch, thread_rows, ci):
    """ILU(0) factorisation with one warp per row (default) and one thread
    per row (PSCU_FACTOR_THREAD): factors bit-identical to ilu0.hpp."""
    if thread_rows == "1":
        monkeypatch.setenv("PSCU_FACTOR_THREAD", "1")
    s = O.RefSystem(**PLAN_CASES[ci])
    a = s.csr()
    ri = O.RefIlu(O.RefCsr(a))
    ilu = S.Ilu0(S.CsrMatrix(a.row_ptr, a.cols, a.vals))
    assert same(ilu.factors(), ri.factors())


@pytest.mark.parametrize("pad", ["0", "1"])
@pytest.mark.parametrize("persist,flow", [("0", "0"), ("1", "0"), ("0", "1"), ("0", "2")])
def test_ilu0_persistent_levels_bitwise(S, monkeypatch, pad, persist, flow):
    """Task-level plans swept by one cooperative launch per sweep (grid
    barrier between task levels, PSCU_LEVEL_PERSIST; or barrier-free
    dataflow waits on the sources, PSCU_LEVEL_FLOW) or per-level launches,
    with and without the 8-entry row padding (PSCU_LEVEL_PAD, cached per
    process: a fresh process per variant); byte-level comparison."""
    import subprocess, sys, os
    code = r'''
import sys, numpy as np
sys.path.insert(0, "tests")
import oracle_ref as O
from paper_2009_13840_b200 import solver as S
for c in [dict(mesh="unit-tri", n=12, jitter=0.2, seed=0, side="top", scheme="hho-dp", strategy="v-cond", k=3, data="sincos"),
          dict(family="trapz", n=6, scheme="hho-dp", strategy="vp-cond", k=2)]:
    s = O.RefSystem(**c); a = s.csr(); ri = O.RefIlu(O.RefCsr(a))
    ilu = S.Ilu0(S.CsrMatrix(a.row_ptr, a.cols, a.vals))
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert ilu.apply(x).tobytes() == ri.apply(x).tobytes()
print("persistent ok")
'''
    env = dict(os.environ, PSCU_LEVEL_PERSIST=persist, PSCU_WALK_MODE="levels",
               PSCU_LEVEL_PERSIST_MIN_ROWS="0", PSCU_LEVEL_PAD=pad, PSCU_LEVEL_FLOW=flow)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "persistent ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("mode", ["default", "levels"])
def test_ilu0_oversize_tasks_bitwise(S, monkeypatch, mode):
    """Rows longer than the warp kernel's task buffers (walk.cu level_chunk:
    kLevelMaxNz entries) fall back to the thread-per-task kernel and keep
    the (default-on) persistent sweep off (advisor finding, round 1)."""
    if mode != "default":
        monkeypatch.setenv("PSCU_WALK_MODE", mode)
    monkeypatch.setenv("PSCU_LEVEL_PERSIST_MIN_ROWS", "0")
    a = synthetic.long_row_csr()
    ri = O.RefIlu(O.RefCsr(a))
    ilu = S.Ilu0(S.CsrMatrix(a.row_ptr, a.cols, a.vals))
    assert ilu.factors().tobytes() == ri.factors().tobytes()
    for seed in range(2):
        x = np.random.default_rng(seed).standard_normal(a.n)
        assert ilu.apply(x).tobytes() == ri.apply(x).tobytes()


def _banded(n, seed):
    """Diagonally dominant banded CSR (columns i-3, i-1, i, i+1, i+5):
    a cheap stand-in with the coarse level's size for Krylov parity."""
    rng = np.random.default_rng(seed)
    offs = np.array([-3, -1, 0, 1, 5])
    rows = np.repeat(np.arange(n), len(offs))
    cols = (rows.reshape(n, -1) + offs).ravel()
    keep = (cols >= 0) & (cols < n)
    rows, cols = rows[keep], cols[keep]
    vals = rng.uniform(-1.0, 1.0, len(cols))
    vals[rows == cols] = 3.0 + rng.uniform(0.0, 1.0, n)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return O.Csr(np.cumsum(rp), cols.astype(np.int32), vals)


@pytest.mark.parametrize("n,force", [(400_000, "1"), (3_194_880, "0")],
                         ids=["forced-400k", "config5-coarse-size"])
def test_gmres_smem_arnoldi_bitwise(S, monkeypatch, n, force):
    """The shared-memory Arnoldi step (arnoldi_smem_kernel: w resident in
    shared memory, 2048 lanes per CTA, basis vectors streamed through L2):
    forced at 400 k unknowns, and at the config-5 coarse size (3,194,880:
    2^18 lanes, 13 elements per lane, 128 CTAs) where it is the production
    path. Unpreconditioned GMRES (the banded matrix's ILU(0) would be one
    sequential chain), bitwise against the reference."""
    monkeypatch.setenv("PSCU_MGS_FORCE_SMEM", force)
    a = _banded(n, 3)
    ra = O.RefCsr(a)
    m = S.CsrMatrix(a.row_ptr, a.cols, a.vals)
    rng = np.random.default_rng(9)
    b = rng.standard_normal(n)
    x0 = rng.standard_normal(n)
    maxit = 40 if n < 1_000_000 else 24
    r = O.ref_gmres(ra, None, b, x0, maxit, 0.0)
    g = S.gmres(m, None, b, x0, maxit, 0.0)
    assert g.iterations == r["its"] and g.rel_residual == r["rel"]
    assert same(g.x, r["x"])
