"""Device post-processing: StokesSystem::recover_solution
(assemble.hpp:58-66) and error_norms (errors.hpp:32-117) through the product
path (host point tables -> pscu_recover_batch -> pscu_error_accumulate),
against the unmodified reference's recover_solution + error_norms on the
same global vector. Bitwise: the recovered local vectors and all four norms,
across batch boundaries (the reference sums each integral in one sequential
chain over elements, which the device reproduces batch by batch)."""
import numpy as np
import pytest

import oracle_ref as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="no oracle")]


@pytest.fixture(scope="module")
def H():
    from paper_2009_13840_b200 import build, host
    build.build_host()
    return host


CASES = [
    # (mesh kind / family, n, scheme, strategy, k, data, x source, batch)
    ("unit-quad", 8, "hho-dp", "v-cond", 1, "sincos", "solve", 7),
    ("unit-tri", 6, "hho-dp", "vp-cond", 3, "sincos", "random", 1000),
    ("tri", 3, "hho-hp", "vp-cond", 2, "exp", "random", 5),
    ("trapz", 3, "hho-hp", "uncond", 1, "exp", "solve", 4),
    ("trapz", 2, "hho-dp", "v-cond", 4, "exp", "random", 3),  # nrec 21: two-lane dots
]


def _systems(H, kind, n, scheme, strat, k, data):
    if kind.startswith("unit-"):
        tri = kind == "unit-tri"
        ref = O.RefSystem(mesh=kind, n=n, seed=0, jitter=0.2, side="top", scheme=scheme,
                          strategy=strat, k=k, data=data)
        mesh = H.Mesh.unit_square(n, tri=tri, jitter=0.2, seed=0, neumann="top")
    else:
        ref = O.RefSystem(family=kind, n=n, scheme=scheme, strategy=strat, k=k, data=data)
        mesh = H.Mesh.family(kind, n, neumann="right")
    return ref, H.LocalSystem(mesh, scheme, strat, k, data=data)


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[2]}-{c[3]}-k{c[4]}" for c in CASES])
def test_error_norms_bitwise(H, case):
    kind, n, scheme, strat, k, data, xsrc, batch = case
    ref, loc = _systems(H, kind, n, scheme, strat, k, data)
    A, b, rec = H.assemble_stokes(loc, recovery=True)
    assert b.tobytes() == ref.rhs().tobytes()
    if xsrc == "solve":
        x = ref.solve([k], coarse="lu", rtol=1e-10)["x"]
    else:
        x = np.random.default_rng(11).standard_normal(ref.n)
    want, want_loc = ref.error_norms(x, data, nloc=loc.n_local)
    got, got_loc = H.error_norms(loc, x, rec, batch=batch, return_locals=True)
    assert got_loc.tobytes() == want_loc.tobytes()
    assert got.as_array().tobytes() == want.tobytes(), (got, want)
    if xsrc == "solve":
        assert 0 < got.u < 1 and np.isfinite(got.as_array()).all()

