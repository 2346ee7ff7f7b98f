"""Host point tables of the device error norms (psh_error_tables, SURVEY.md
§8(f)4), checked on the CPU: a float-by-float restatement of the device
kernel (paper_2009_13840_b200/csrc/errors.cu, itself a restatement of
errors.hpp:32-117) run over the tables and the reference's own recovered
local vectors reproduces the reference's error_norms bit for bit — so the
tables carry exactly the reference's reconstruction, basis values,
quadrature and closed-form field. Plus the argument checks."""
import math

import numpy as np
import pytest

import oracle_ref as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="no oracle")


@pytest.fixture(scope="module")
def H():
    from paper_2009_13840_b200 import build, host
    build.build_host()
    return host


def _rdot(x, y):
    """include/eigen_subset repro_dot (T lanes, pairwise lane tree)."""
    n = len(x)
    T = 1
    while T < (n + 15) // 16:
        T *= 2
    part = [0.0] * T
    for i in range(n):
        part[i % T] = part[i % T] + float(x[i]) * float(y[i])
    while T > 1:
        part = [part[2 * k] + part[2 * k + 1] for k in range(T // 2)]
        T //= 2
    return part[0]


def _norms(dims, tab, locs):
    nrec, ns, nq, qs, per, ne, nf, npr, nloc, nfc, hyb = (int(v) for v in dims)
    acc = [0.0, 0.0, 0.0, 0.0]
    for e, x in enumerate(locs):
        t = tab[e * per:(e + 1) * per]
        P = t[:nrec * ns].reshape(ns, nrec).T
        comp = np.zeros((ns, 2))
        for c in range(2):
            comp[:ne, c] = x[c * ne:(c + 1) * ne]
            for lf in range(nfc):
                o = 2 * ne + lf * 2 * nf + c * nf
                comp[ne + lf * nf:ne + (lf + 1) * nf, c] = x[o:o + nf]
        gco = np.zeros((nrec, 2))
        for c in range(2):
            for i in range(nrec):
                s = 0.0
                for kk in range(ns):
                    s = s + float(P[i, kk]) * float(comp[kk, c])
                gco[i, c] = s
        uco = np.zeros((nrec, 2))
        if hyb:
            uco[:ne] = comp[:ne]
        else:
            uco[:] = gco
        pco = np.zeros(nrec)
        off = 2 * (ne + nfc * nf)
        pco[:npr] = x[off:off + npr]
        for q in range(nq):
            r = t[nrec * ns + q * qs:nrec * ns + (q + 1) * qs]
            w, v = float(r[0]), r[1:1 + nrec]
            g = (r[1 + nrec:1 + 2 * nrec], r[1 + 2 * nrec:1 + 3 * nrec])
            ex = r[1 + 3 * nrec:]
            div = 0.0
            for c in range(2):
                du = _rdot(v, uco[:, c]) - float(ex[c])
                acc[0] = acc[0] + w * du * du
                for d in range(2):
                    dg = _rdot(g[d], gco[:, c]) - float(ex[2 + 2 * c + d])
                    acc[1] = acc[1] + w * dg * dg
                div = div + _rdot(g[c], uco[:, c])
            dp = _rdot(v, pco) - float(ex[6])
            acc[2] = acc[2] + w * dp * dp
            acc[3] = acc[3] + w * div * div
    return np.array([math.sqrt(a) for a in acc])


@pytest.mark.parametrize("case", [("tri", 2, "hho-hp", "vp-cond", 1, "exp"),
                                  ("unit-quad", 3, "hho-dp", "v-cond", 2, "sincos")],
                         ids=["tri-hp-k1", "quad-dp-k2"])
def test_tables_reproduce_reference_error_norms(H, case):
    kind, n, scheme, strat, k, data = case
    if kind.startswith("unit-"):
        ref = O.RefSystem(mesh=kind, n=n, seed=0, jitter=0.2, side="top", scheme=scheme,
                          strategy=strat, k=k, data=data)
        mesh = H.Mesh.unit_square(n, jitter=0.2, seed=0, neumann="top")
    else:
        ref = O.RefSystem(family=kind, n=n, scheme=scheme, strategy=strat, k=k, data=data)
        mesh = H.Mesh.family(kind, n, neumann="right")
    loc = H.LocalSystem(mesh, scheme, strat, k, data=data)
    x = np.random.default_rng(3).standard_normal(ref.n)
    want, locs = ref.error_norms(x, data, nloc=loc.n_local)
    dims, tab = H.error_tables(loc)
    assert int(dims[8]) == loc.n_local and len(tab) == loc.nelem * int(dims[4])
    # the weights integrate the element areas: the unit-square / family domain
    w = sum(tab[e * int(dims[4]) + int(dims[0]) * int(dims[1]) + q * int(dims[3])]
            for e in range(loc.nelem) for q in range(int(dims[2])))
    assert w == pytest.approx(1.0 if kind.startswith("unit-") else 4.0, rel=1e-12)
    # tables for a sub-range equal the slice of the full tables
    _, sub = H.error_tables(loc, 1, 2)
    per = int(dims[4])
    assert sub.tobytes() == tab[per:3 * per].tobytes()
    got = _norms(dims, tab, locs)
    assert got.tobytes() == want.tobytes(), (got, want)


def test_error_tables_reject_bad_input(H):
    mesh = H.Mesh.unit_square(2)
    loc = H.LocalSystem(mesh, "hho-dp", "v-cond", 1, data="zero")
    with pytest.raises(ValueError, match="closed form"):
        H.error_tables(loc)
    loc = H.LocalSystem(mesh, "hho-dp", "v-cond", 1, data="sincos")
    with pytest.raises(ValueError, match="out of bounds"):
        H.error_tables(loc, 3, 5)
