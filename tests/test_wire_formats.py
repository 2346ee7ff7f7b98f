"""Wire formats on the CPU against the unmodified
reference: pmesh2 v1 mesh files (write_mesh / read_mesh, mesh.hpp:535-645)
and the MatrixMarket export of the assembled operator
(write_matrix_market, csr.hpp:98-111), byte for byte; the reader's error
behaviour (std::runtime_error with the reference's messages)."""
import os

import numpy as np
import pytest

import oracle_ref as O
from paper_2009_13840_b200 import build, host

pytestmark = pytest.mark.skipif(not (O.ref_available() and os.path.exists(O.WIRE)),
                                reason="reference oracle not built")


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build_host()


MESHES = [dict(kind="unit-tri", n=8, jitter=0.2, side="top"),
          dict(kind="unit-quad", n=6, jitter=0.0, side="top"),
          dict(kind="family", family="trapz", n=4, side="right")]


class _Ref:
    def __init__(self, c):
        self.c = c

    def write_mesh(self, path):
        c = self.c
        O.ref_write_mesh(path, kind=c["kind"], family=c.get("family", "trapz"), n=c["n"],
                         jitter=c.get("jitter", 0.0), side=c["side"])


def _pair(c):
    if c["kind"] == "family":
        ours = host.Mesh.family(c["family"], c["n"], neumann=c["side"])
    else:
        ours = host.Mesh.unit_square(c["n"], tri=c["kind"] == "unit-tri", jitter=c["jitter"],
                                     seed=0, neumann=c["side"])
    return _Ref(c), ours


@pytest.mark.parametrize("c", MESHES, ids=[m["kind"] for m in MESHES])
def test_mesh_write_matches_reference(tmp_path, c):
    ref, ours = _pair(c)
    a, b = tmp_path / "ref.pmesh", tmp_path / "ours.pmesh"
    ref.write_mesh(str(a))
    ours.write(str(b))
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.parametrize("c", MESHES, ids=[m["kind"] for m in MESHES])
def test_mesh_read_roundtrip(tmp_path, c):
    ref, ours = _pair(c)
    src = tmp_path / "ref.pmesh"
    ref.write_mesh(str(src))
    m = host.Mesh.read(str(src))
    assert np.array_equal(m.faces(), ours.faces()) and np.array_equal(m.vertices(), ours.vertices())
    back, ref_back = tmp_path / "back.pmesh", tmp_path / "ref_back.pmesh"
    m.write(str(back))
    O.ref_mesh_roundtrip(str(src), str(ref_back))
    assert back.read_bytes() == src.read_bytes() == ref_back.read_bytes()
    # nf = 0: the faces are derived (first-seen, boundary Dirichlet) like the reference
    lines = src.read_text().splitlines()
    hdr = lines[0].split()
    nf = int(hdr[4])
    derived = tmp_path / "derived.pmesh"
    derived.write_text("\n".join([" ".join(hdr[:4] + ["0"])] + lines[1:len(lines) - nf]) + "\n")
    d_ours, d_ref = tmp_path / "d_ours.pmesh", tmp_path / "d_ref.pmesh"
    host.Mesh.read(str(derived)).write(str(d_ours))
    O.ref_mesh_roundtrip(str(derived), str(d_ref))
    assert d_ours.read_bytes() == d_ref.read_bytes()


BAD = [("pmesh3 v1 3 1 0\n", "line 1: malformed header"),
       ("pmesh2 v1 3 0 0\n", "line 1: no elements"),
       ("pmesh2 v1 3 1 0\nv 0 0\nv 1 0\ne 0 1 2\n", "expected a 'v' record"),
       ("pmesh2 v1 3 1 0\nv 0 0\nv 1 0\nv 0 1\ne 0 1 5\n", "vertex index 5 out of range"),
       ("pmesh2 v1 3 1 0\nv 0 0\nv 1 0\nv 0 1\ne 0 1\n", "fewer than 3 vertices"),
       ("pmesh2 v1 3 1 1\nv 0 0\nv 1 0\nv 0 1\ne 0 1 2\nf 0 1 0 -1 i\n",
        "boundary face tagged interior"),
       ("pmesh2 v1 3 1 1\nv 0 0\nv 1 0\nv 0 1\ne 0 1 2\nf 0 1 0 -1 x\n", "unknown face tag")]


@pytest.mark.parametrize("text,msg", BAD)
def test_mesh_reader_rejects_like_reference(tmp_path, text, msg):
    p = tmp_path / "bad.pmesh"
    p.write_text(text)
    with pytest.raises(RuntimeError) as ours:
        host.Mesh.read(str(p))
    with pytest.raises(RuntimeError) as ref:
        O.ref_mesh_roundtrip(str(p), str(tmp_path / "x.pmesh"))
    assert msg in str(ours.value) and str(ours.value) == str(ref.value)


@pytest.mark.parametrize("scheme,strategy,k", [("hho-dp", "v-cond", 2), ("hho-hp", "vp-cond", 1),
                                               ("dg", "uncond", 1)])
def test_matrix_market_matches_reference(tmp_path, scheme, strategy, k):
    ref = O.RefSystem(family="trapz", n=3, scheme=scheme, strategy=strategy, k=k)
    a = ref.csr()
    p1, p2 = tmp_path / "ref.mtx", tmp_path / "ours.mtx"
    O.ref_write_matrix_market(str(p1), family="trapz", n=3, scheme=scheme, strategy=strategy, k=k)
    host.write_matrix_market(a.row_ptr, a.cols, a.vals, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
