"""End-to-end product pipeline on the GPU: host local blocks -> device
condensation + assembly -> device hierarchy + FGMRES, against the
reference. The device condensation and assembly are bit-exact on the
reference's own local blocks, and the product's own host producer builds
those blocks bit for bit, so the whole product pipeline is bitwise."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle_ref as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="no oracle")]


@pytest.fixture(scope="module")
def M():
    from paper_2009_13840_b200 import build, host, solver, _native
    build.build_host()
    return host, solver, _native


def test_device_condense_assemble_bitwise_on_reference_blocks(M, tmp_path):
    host, S, N = M
    for fam, scheme, strat, k in [("trapz", "hho-dp", "v-cond", 3), ("tri", "hho-hp", "vp-cond", 2),
                                  ("trapz", "hho-dp", "vp-cond", 2)]:
        ref = O.RefSystem(family=fam, n=3, scheme=scheme, strategy=strat, k=k, data="exp")
        a = ref.csr()
        ne = ref.layout.n_elements
        mats, rhss, kept = [], [], []
        for e in range(ne):
            m, r, elim = ref.local_blocks(e, data="exp")
            mats.append(np.asfortranarray(m).ravel(order="F"))
            rhss.append(r)
            kept.append(ref.condensation(e)["kept_global"])
        mats = np.ascontiguousarray(np.concatenate(mats))
        rhss = np.ascontiguousarray(np.concatenate(rhss))
        kept = np.ascontiguousarray(np.concatenate(kept))
        elim = np.ascontiguousarray(elim, np.int32)
        n_local = int(np.sqrt(len(mats) // ne))
        L = ref.layout
        lay = S.make_layout(L.scheme, L.strategy, L.k, L.n_faces, L.n_elements)
        ctx = S.default_context()
        h = C.c_void_p()
        rhs = np.zeros(a.n)
        N.check(ctx.lib.pscu_condense_assemble(ctx.h, ne, n_local, mats.ctypes.data,
                                               rhss.ctypes.data, len(elim), elim.ctypes.data,
                                               kept.ctypes.data, a.n, a.row_ptr.ctypes.data,
                                               a.cols.ctypes.data, C.byref(lay), N.PSCU_HOST,
                                               C.byref(h), rhs.ctypes.data, None, None))
        m = S.CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
        m._owned = True
        rp, cl, vl = m.download()
        assert np.all(vl == a.vals) and np.all(cl == a.cols)
        assert np.all(rhs == ref.rhs())
        if os.path.exists(O.WIRE):
            # the pattern-parity wire format (csr.hpp:98-111), byte for byte
            p1, p2 = tmp_path / "ref.mtx", tmp_path / "dev.mtx"
            O.ref_write_matrix_market(str(p1), family=fam, n=3, scheme=scheme, strategy=strat, k=k)
            host.write_matrix_market(rp, cl, vl, str(p2))
            assert p1.read_bytes() == p2.read_bytes()


@pytest.mark.parametrize("case", [
    dict(kind="unit-quad", n=16, tri=False, jitter=0.0, k=1, strat="v-cond", deg=[1, 0]),
    dict(kind="unit-tri", n=16, tri=True, jitter=0.2, k=3, strat="v-cond", deg=[3, 2, 1, 0]),
    dict(kind="unit-tri", n=8, tri=True, jitter=0.2, k=3, strat="vp-cond", deg=[3, 2, 1, 0]),
], ids=["config1", "config2a-16", "config2b-8"])
def test_product_pipeline_matches_reference(M, case):
    host, S, N = M
    ref = O.RefSystem(mesh=case["kind"], n=case["n"], seed=0, jitter=case["jitter"], side="top",
                      scheme="hho-dp", strategy=case["strat"], k=case["k"], data="sincos")
    mesh = host.Mesh.unit_square(case["n"], tri=case["tri"], jitter=case["jitter"], seed=0,
                                 neumann="top")
    loc = host.LocalSystem(mesh, "hho-dp", case["strat"], case["k"], data="sincos")
    A, b = host.assemble_stokes(loc)
    a = ref.csr()
    rp, cl, vl = A.download()
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(cl, a.cols)
    assert vl.tobytes() == a.vals.tobytes()
    assert b.tobytes() == ref.rhs().tobytes()
    r = ref.solve(case["deg"], coarse="gmres-ilu", rtol=1e-8, restart=30)
    cfg = S.LevelConfig(degrees=case["deg"], coarse="gmres-ilu", outer_rtol=1e-8, restart=30)
    h = S.LevelHierarchy(A, loc.layout(), cfg)
    x, hist, rep = h.solve(b)
    assert rep.converged and rep.outer_its == r["its"] and rep.coarse_its == r["coarse_its"]
    assert hist.tobytes() == r["hist"].tobytes() and x.tobytes() == r["x"].tobytes()
