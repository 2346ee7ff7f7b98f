"""ctypes bindings to the oracles (TEST INFRASTRUCTURE ONLY).

* ``Ref*``   — oracle/_ref/libpstokes_ref.so: the UNMODIFIED reference headers
  compiled against include/eigen_subset (oracle/Makefile, oracle/ref_driver.cpp).
* ``Port*``  — oracle/_build/libpstokes_oracle.so: the plain-C restatement.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs import this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpstokes_ref.so")
PORT_SO = os.path.join(ROOT, "oracle", "_build", "libpstokes_oracle.so")

SCHEMES = {"hho-dp": 0, "hho-hp": 1, "dg": 2}
STRATEGIES = {"uncond": 0, "v-cond": 1, "vp-cond": 2}
SIDES = {"left": 0, "right": 1, "top": 2, "bottom": 3}
DATA = {"zero": 0, "exp": 1, "sincos": 2}
MESH_KINDS = {"family": 0, "unit-quad": 1, "unit-tri": 2}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_ref = None
_port = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def port_available() -> bool:
    return os.path.exists(PORT_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_system_create.restype = vp
        lib.ref_system_create.argtypes = [C.c_int, C.c_char_p, C.c_int, C.c_ulonglong, C.c_double,
                                          C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
        lib.ref_system_destroy.argtypes = [vp]
        for f in ("ref_system_dim", "ref_system_nnz"):
            getattr(lib, f).restype = C.c_longlong
            getattr(lib, f).argtypes = [vp]
        lib.ref_system_t_assembly.restype = C.c_double
        lib.ref_system_t_assembly.argtypes = [vp]
        lib.ref_system_csr.argtypes = [vp, _i64p, _i32p, _f64p]
        lib.ref_system_rhs.argtypes = [vp, _f64p]
        lib.ref_system_layout.argtypes = [vp, _i32p]
        lib.ref_mesh_sizes.argtypes = [vp, _i64p]
        lib.ref_mesh_export.argtypes = [vp, _f64p, _i64p, _i32p, _i32p, _i32p, _i32p]
        lib.ref_local_element.argtypes = [vp, C.c_int, _i32p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_local_blocks.argtypes = [vp, C.c_int, C.c_int, _i32p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        lib.ref_csr_create.restype = vp
        lib.ref_csr_create.argtypes = [C.c_int, _i64p, _i32p, _f64p]
        lib.ref_csr_destroy.argtypes = [vp]
        lib.ref_csr_multiply.argtypes = [vp, _f64p, _f64p]
        lib.ref_ilu_create.restype = vp
        lib.ref_ilu_create.argtypes = [vp]
        lib.ref_ilu_destroy.argtypes = [vp]
        lib.ref_ilu_apply.argtypes = [vp, _f64p, _f64p]
        lib.ref_ilu_factors.argtypes = [vp, _f64p]
        lib.ref_gmres.argtypes = [vp, vp, _f64p, _f64p, C.c_int, C.c_double, C.c_int, _f64p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int)]
        lib.ref_fgmres.argtypes = [vp, vp, _f64p, C.c_int, C.c_double, _f64p, C.POINTER(C.c_int),
                                   C.POINTER(C.c_double), C.POINTER(C.c_int)]
        lib.ref_hier_create.restype = vp
        lib.ref_hier_create.argtypes = [vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        lib.ref_hier_destroy.argtypes = [vp]
        lib.ref_hier_nlev.argtypes = [vp]
        lib.ref_hier_t_setup.restype = C.c_double
        lib.ref_hier_t_setup.argtypes = [vp]
        for f in ("ref_hier_level_dim", "ref_hier_level_nnz"):
            getattr(lib, f).restype = C.c_longlong
            getattr(lib, f).argtypes = [vp, C.c_int]
        lib.ref_hier_level_csr.argtypes = [vp, C.c_int, _i64p, _i32p, _f64p]
        lib.ref_hier_level_downmap.restype = C.c_longlong
        lib.ref_hier_level_downmap.argtypes = [vp, C.c_int, C.c_void_p]
        lib.ref_hier_level_ilu.argtypes = [vp, C.c_int, _f64p]
        lib.ref_hier_vcycle.argtypes = [vp, C.c_int, _f64p, _f64p]
        lib.ref_hier_coarse_its.restype = C.c_longlong
        lib.ref_hier_coarse_its.argtypes = [vp]
        lib.ref_hier_reset.argtypes = [vp]
        lib.ref_solve.argtypes = [vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  C.c_double, C.c_int, C.c_int, _f64p, C.c_void_p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_int),
                                  C.POINTER(C.c_double), C.POINTER(C.c_int),
                                  C.POINTER(C.c_double)]
        lib.ref_solve_timed.argtypes = [vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_int, C.c_double, C.c_int, C.c_int,
                                        C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int)]
        lib.ref_solve_timed.restype = C.c_int
        lib.ref_solve_system.argtypes = [vp, _i32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                         _f64p, C.POINTER(C.c_int), C.POINTER(C.c_longlong),
                                         C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.POINTER(C.c_int), C.POINTER(C.c_double)]
        lib.ref_inherit.restype = C.c_longlong
        lib.ref_inherit.argtypes = [vp, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p]
        lib.ref_layout_dim.restype = C.c_longlong
        lib.ref_layout_dim.argtypes = [vp, C.c_int]
        lib.ref_error_norms.argtypes = [vp, C.c_int, _f64p, _f64p, C.c_void_p]
        _ref = lib
    return _ref


def _err(lib, fn="ref_last_error"):
    return getattr(lib, fn)().decode()


@dataclass
class Csr:
    row_ptr: np.ndarray  # int64 [n+1]
    cols: np.ndarray  # int32 [nnz]
    vals: np.ndarray  # float64 [nnz]

    @property
    def n(self) -> int:
        return len(self.row_ptr) - 1

    @property
    def nnz(self) -> int:
        return len(self.cols)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        for i in range(self.n):
            s, e = self.row_ptr[i], self.row_ptr[i + 1]
            d[i, self.cols[s:e]] = self.vals[s:e]
        return d


@dataclass
class LayoutInfo:
    scheme: int
    strategy: int
    k: int
    n_faces: int
    n_elements: int
    face_vel: int
    face_press: int
    elem_vel: int
    elem_press: int
    n_vertices: int


class RefSystem:
    """Reference-assembled StokesSystem (assemble_stokes, assemble.hpp:348)."""

    def __init__(self, mesh: str = "family", family: str = "trapz", n: int = 2, seed: int = 1,
                 jitter: float = 0.0, side: str = "right", scheme: str = "hho-dp",
                 strategy: str = "v-cond", k: int = 1, data: str = "exp", eta: float = 0.0):
        lib = ref_lib()
        self.lib = lib
        self.h = lib.ref_system_create(MESH_KINDS[mesh], family.encode(), n, seed, jitter,
                                       SIDES[side], SCHEMES[scheme], STRATEGIES[strategy], k,
                                       DATA[data], eta)
        if not self.h:
            raise RuntimeError(_err(lib))
        self.n = lib.ref_system_dim(self.h)
        self.nnz = lib.ref_system_nnz(self.h)
        lay = np.zeros(10, np.int32)
        lib.ref_system_layout(self.h, lay)
        self.layout = LayoutInfo(*[int(v) for v in lay])

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_system_destroy(self.h)
            self.h = None

    def csr(self) -> Csr:
        rp = np.zeros(self.n + 1, np.int64)
        cols = np.zeros(self.nnz, np.int32)
        vals = np.zeros(self.nnz, np.float64)
        self.lib.ref_system_csr(self.h, rp, cols, vals)
        return Csr(rp, cols, vals)

    def rhs(self) -> np.ndarray:
        r = np.zeros(self.n, np.float64)
        self.lib.ref_system_rhs(self.h, r)
        return r

    def mesh(self):
        sz = np.zeros(4, np.int64)
        self.lib.ref_mesh_sizes(self.h, sz)
        nv, ne, nf, nl = (int(v) for v in sz)
        xy = np.zeros(2 * nv)
        eoff = np.zeros(ne + 1, np.int64)
        loops = np.zeros(nl, np.int32)
        faces = np.zeros(5 * nf, np.int32)
        efaces = np.zeros(nl, np.int32)
        esigns = np.zeros(nl, np.int32)
        self.lib.ref_mesh_export(self.h, xy, eoff, loops, faces, efaces, esigns)
        return dict(xy=xy.reshape(nv, 2), eoff=eoff, loops=loops, faces=faces.reshape(nf, 5),
                    efaces=efaces, esigns=esigns)

    def local_blocks(self, e: int, data: str = "exp"):
        sizes = np.zeros(4, np.int32)
        rc = self.lib.ref_local_blocks(self.h, e, DATA[data], sizes, None, None, None)
        if rc:
            raise RuntimeError(_err(self.lib))
        n, ne = int(sizes[0]), int(sizes[1])
        mat = np.zeros(n * n)
        rhs = np.zeros(n)
        elim = np.zeros(max(ne, 1), np.int32)
        self.lib.ref_local_blocks(self.h, e, DATA[data], sizes, mat.ctypes.data, rhs.ctypes.data,
                                  elim.ctypes.data)
        return mat.reshape(n, n, order="F"), rhs, elim[:ne]

    def condensation(self, e: int):
        sizes = np.zeros(4, np.int32)
        rc = self.lib.ref_local_element(self.h, e, sizes, None, None, None, None, None, None)
        if rc:
            raise RuntimeError(_err(self.lib))
        n, ne, nk = (int(v) for v in sizes[:3])
        elim = np.zeros(max(ne, 1), np.int32)
        kept = np.zeros(nk, np.int64)
        schur = np.zeros(nk * nk)
        rr = np.zeros(nk)
        coup = np.zeros(max(ne * nk, 1))
        er = np.zeros(max(ne, 1))
        self.lib.ref_local_element(self.h, e, sizes, elim.ctypes.data, kept.ctypes.data,
                                   schur.ctypes.data, rr.ctypes.data, coup.ctypes.data,
                                   er.ctypes.data)
        return dict(elim=elim[:ne], kept_global=kept, schur=schur.reshape(nk, nk, order="F"),
                    reduced_rhs=rr, elim_coupling=coup[: ne * nk].reshape(ne, nk, order="F"),
                    elim_rhs=er[:ne])

    def layout_dim(self, k: int) -> int:
        return int(self.lib.ref_layout_dim(self.h, k))

    def inherit(self, kf: int, kc: int):
        nnz = self.lib.ref_inherit(self.h, kf, kc, None, None, None, None)
        if nnz < 0:
            raise RuntimeError(_err(self.lib))
        nc = self.layout_dim(kc)
        rp = np.zeros(nc + 1, np.int64)
        cols = np.zeros(nnz, np.int32)
        vals = np.zeros(nnz)
        c2f = np.zeros(nc, np.int64)
        self.lib.ref_inherit(self.h, kf, kc, rp.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                             c2f.ctypes.data)
        return Csr(rp, cols, vals), c2f

    def solve(self, degrees, smoother_iters=2, coarse="gmres-ilu", coarse_rtol=1e-3,
              coarse_maxit=400, rtol=1e-13, maxit=1000, restart=0):
        deg = np.asarray(degrees, np.int32)
        x = np.zeros(self.n)
        hist = np.zeros(maxit + 1)
        its, cits, vcs, rel, conv, ts = (C.c_int(), C.c_longlong(), C.c_int(), C.c_double(),
                                         C.c_int(), C.c_double())
        rc = self.lib.ref_solve(self.h, deg, len(deg), smoother_iters, int(coarse != "lu"),
                                coarse_rtol, coarse_maxit, rtol, maxit, restart, x,
                                hist.ctypes.data, C.byref(its), C.byref(cits), C.byref(vcs),
                                C.byref(rel), C.byref(conv), C.byref(ts))
        if rc:
            raise RuntimeError(_err(self.lib))
        return dict(x=x, hist=hist[: its.value].copy(), its=its.value, coarse_its=cits.value,
                    vcycles=vcs.value, rel=rel.value, converged=bool(conv.value), t_solve=ts.value)

    def error_norms(self, x, data: str, nloc: int = 0):
        """recover_solution (assemble.hpp:58-66) + error_norms (errors.hpp:32-117)
        of the global vector x: {u, grad_u, p, div_u}, plus the recovered local
        vectors (n_elements x nloc) when nloc is given."""
        out = np.zeros(4)
        loc = np.zeros((self.layout.n_elements, nloc)) if nloc else None
        rc = self.lib.ref_error_norms(self.h, DATA[data], np.ascontiguousarray(x, np.float64), out,
                                      loc.ctypes.data if nloc else None)
        if rc:
            raise RuntimeError(_err(self.lib))
        return (out, loc) if nloc else out

    def solve_timed(self, degrees, maxit, smoother_iters=2, coarse="gmres-ilu", coarse_rtol=1e-3,
                    coarse_maxit=400, rtol=1e-8, restart=0):
        """Reference hierarchy setup time and per-iteration end times of the
        first `maxit` FGMRES iterations (bench.py's reference arm)."""
        deg = np.asarray(degrees, np.int32)
        stamps = np.zeros(maxit + 1)
        t_setup, its = C.c_double(), C.c_int()
        rc = self.lib.ref_solve_timed(self.h, deg.ctypes.data, len(deg), smoother_iters,
                                      int(coarse != "lu"), C.c_double(coarse_rtol), coarse_maxit,
                                      C.c_double(rtol), maxit, restart, C.byref(t_setup),
                                      stamps.ctypes.data, C.byref(its))
        if rc:
            raise RuntimeError(_err(self.lib))
        return t_setup.value, stamps[: its.value].copy()

    def solve_system(self, degrees, smoother_iters=2, coarse="lu", rtol=1e-13, maxit=1000):
        deg = np.asarray(degrees, np.int32)
        x = np.zeros(self.n)
        its, cits, vcs, rel, conv, ts = (C.c_int(), C.c_longlong(), C.c_int(), C.c_double(),
                                         C.c_int(), C.c_double())
        rc = self.lib.ref_solve_system(self.h, deg, len(deg), smoother_iters, int(coarse != "lu"),
                                       rtol, maxit, x, C.byref(its), C.byref(cits), C.byref(vcs),
                                       C.byref(rel), C.byref(conv), C.byref(ts))
        if rc:
            raise RuntimeError(_err(self.lib))
        return dict(x=x, its=its.value, coarse_its=cits.value, vcycles=vcs.value, rel=rel.value,
                    converged=bool(conv.value), t_solve=ts.value)


class RefHierarchy:
    """LevelHierarchy (plevels.hpp:115-212) built by the reference."""

    def __init__(self, sysobj: RefSystem, degrees, smoother_iters=2, coarse="gmres-ilu",
                 coarse_rtol=1e-3, coarse_maxit=400):
        self.lib = sysobj.lib
        self.sys = sysobj
        deg = np.asarray(degrees, np.int32)
        self.h = self.lib.ref_hier_create(sysobj.h, deg, len(deg), smoother_iters,
                                          int(coarse != "lu"), coarse_rtol, coarse_maxit)
        if not self.h:
            raise RuntimeError(_err(self.lib))
        self.nlev = self.lib.ref_hier_nlev(self.h)
        self.t_setup = self.lib.ref_hier_t_setup(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_hier_destroy(self.h)
            self.h = None

    def level_csr(self, l: int) -> Csr:
        n = self.lib.ref_hier_level_dim(self.h, l)
        nnz = self.lib.ref_hier_level_nnz(self.h, l)
        rp = np.zeros(n + 1, np.int64)
        cols = np.zeros(nnz, np.int32)
        vals = np.zeros(nnz)
        self.lib.ref_hier_level_csr(self.h, l, rp, cols, vals)
        return Csr(rp, cols, vals)

    def down_map(self, l: int) -> np.ndarray:
        m = self.lib.ref_hier_level_downmap(self.h, l, None)
        out = np.zeros(m, np.int64)
        if m:
            self.lib.ref_hier_level_downmap(self.h, l, out.ctypes.data)
        return out

    def level_ilu(self, l: int) -> np.ndarray:
        nnz = self.lib.ref_hier_level_nnz(self.h, l)
        lu = np.zeros(nnz)
        if self.lib.ref_hier_level_ilu(self.h, l, lu):
            raise RuntimeError("level has no ILU factor")
        return lu

    def vcycle(self, l: int, d: np.ndarray) -> np.ndarray:
        d = np.ascontiguousarray(d, np.float64)
        c = np.zeros_like(d)
        if self.lib.ref_hier_vcycle(self.h, l, d, c):
            raise RuntimeError(_err(self.lib))
        return c

    def coarse_its(self) -> int:
        return int(self.lib.ref_hier_coarse_its(self.h))

    def reset(self):
        self.lib.ref_hier_reset(self.h)


class RefCsr:
    def __init__(self, a: Csr):
        self.lib = ref_lib()
        self.a = a
        self.h = self.lib.ref_csr_create(a.n, a.row_ptr, a.cols, a.vals)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_csr_destroy(self.h)

    def multiply(self, x):
        y = np.zeros(self.a.n)
        self.lib.ref_csr_multiply(self.h, np.ascontiguousarray(x, np.float64), y)
        return y


class RefIlu:
    def __init__(self, a: RefCsr):
        self.lib = a.lib
        self.a = a
        self.h = self.lib.ref_ilu_create(a.h)
        if not self.h:
            raise RuntimeError(_err(self.lib))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_ilu_destroy(self.h)

    def apply(self, x):
        y = np.zeros(self.a.a.n)
        self.lib.ref_ilu_apply(self.h, np.ascontiguousarray(x, np.float64), y)
        return y

    def factors(self):
        lu = np.zeros(self.a.a.nnz)
        self.lib.ref_ilu_factors(self.h, lu)
        return lu


def ref_gmres(a: RefCsr, ilu, rhs, x0, max_it, rtol, left=False):
    lib = a.lib
    x = np.zeros(a.a.n)
    its, rel, conv = C.c_int(), C.c_double(), C.c_int()
    rc = lib.ref_gmres(a.h, ilu.h if ilu else None, np.ascontiguousarray(rhs, np.float64),
                       np.ascontiguousarray(x0, np.float64), max_it, rtol, int(left), x,
                       C.byref(its), C.byref(rel), C.byref(conv))
    if rc:
        raise RuntimeError(_err(lib))
    return dict(x=x, its=its.value, rel=rel.value, converged=bool(conv.value))


def ref_fgmres(a: RefCsr, ilu, rhs, max_it, rtol):
    lib = a.lib
    x = np.zeros(a.a.n)
    its, rel, conv = C.c_int(), C.c_double(), C.c_int()
    rc = lib.ref_fgmres(a.h, ilu.h if ilu else None, np.ascontiguousarray(rhs, np.float64),
                        max_it, rtol, x, C.byref(its), C.byref(rel), C.byref(conv))
    if rc:
        raise RuntimeError(_err(lib))
    return dict(x=x, its=its.value, rel=rel.value, converged=bool(conv.value))


# ---------------------------------------------------------------------------
# plain-C restatement
# ---------------------------------------------------------------------------

class _PoCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("row_ptr", C.c_void_p), ("cols", C.c_void_p),
                ("vals", C.c_void_p)]


class PoLayout(C.Structure):
    _fields_ = [(f, C.c_int) for f in ("scheme", "strategy", "k", "n_faces", "n_elements",
                                       "face_vel", "face_press", "elem_vel", "elem_press",
                                       "dim")]


def port_lib():
    global _port
    if _port is None:
        lib = C.CDLL(PORT_SO)
        vp = C.c_void_p
        lib.po_last_error.restype = C.c_char_p
        lib.po_make_layout.argtypes = [C.c_int] * 5 + [C.POINTER(PoLayout)]
        lib.po_make_layout3.argtypes = [C.c_int] * 5 + [C.POINTER(PoLayout)]
        lib.po_condense_assemble.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, vp, vp,
                                             C.POINTER(PoLayout), C.POINTER(_PoCsr), vp, vp]
        lib.po_layout_dim.restype = C.c_int64
        lib.po_layout_dim.argtypes = [C.POINTER(PoLayout)]
        lib.po_coarse_to_fine_map.argtypes = [C.POINTER(PoLayout), C.POINTER(PoLayout), _i64p]
        lib.po_dot.restype = C.c_double
        lib.po_dot.argtypes = [_f64p, _f64p, C.c_int64]
        lib.po_csr_multiply.argtypes = [C.POINTER(_PoCsr), _f64p, _f64p]
        lib.po_ilu0_factor.argtypes = [C.POINTER(_PoCsr), _f64p, _i64p]
        lib.po_ilu0_apply.argtypes = [C.POINTER(_PoCsr), _f64p, _i64p, _f64p, _f64p]
        lib.po_inherit.restype = C.c_int64
        lib.po_inherit.argtypes = [C.POINTER(_PoCsr), C.c_int64, _i64p, C.c_int64, vp, vp, vp]
        lib.po_hier_create.restype = vp
        lib.po_hier_create.argtypes = [C.POINTER(_PoCsr), C.POINTER(PoLayout), _i32p, C.c_int,
                                       C.c_int, C.c_double, C.c_int]
        lib.po_hier_create_ex.restype = vp
        lib.po_hier_create_ex.argtypes = [C.POINTER(_PoCsr), C.POINTER(PoLayout), _i32p, C.c_int,
                                          C.c_int, C.c_double, C.c_int, C.c_int]
        lib.po_bj_size.restype = C.c_int64
        lib.po_bj_size.argtypes = [C.POINTER(PoLayout)]
        lib.po_bj_factor.argtypes = [C.POINTER(_PoCsr), C.POINTER(PoLayout), _f64p,
                                     C.POINTER(C.c_int64)]
        lib.po_bj_apply.argtypes = [C.POINTER(PoLayout), _f64p, _f64p, _f64p]
        lib.po_hier_destroy.argtypes = [vp]
        lib.po_hier_level_dim.restype = C.c_int64
        lib.po_hier_level_dim.argtypes = [vp, C.c_int]
        lib.po_hier_level_nnz.restype = C.c_int64
        lib.po_hier_level_nnz.argtypes = [vp, C.c_int]
        lib.po_hier_level_csr.argtypes = [vp, C.c_int, _i64p, _i32p, _f64p]
        lib.po_hier_level_ilu.argtypes = [vp, C.c_int, _f64p]
        lib.po_vcycle.argtypes = [vp, C.c_int, _f64p, _f64p]
        lib.po_hier_coarse_its.restype = C.c_longlong
        lib.po_hier_coarse_its.argtypes = [vp]
        lib.po_solve.argtypes = [vp, _f64p, C.c_double, C.c_int, C.c_int, _f64p, vp,
                                 C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_int),
                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]
        lib.po_condense.argtypes = [C.c_int, _f64p, _f64p, C.c_int, _i32p, _f64p, _f64p, _f64p,
                                    _f64p]
        lib.po_dg_pattern.restype = C.c_int64
        lib.po_dg_pattern.argtypes = [C.POINTER(PoLayout), C.c_int, vp, vp, vp, vp]
        lib.po_dg_assemble.argtypes = [C.POINTER(PoLayout), C.c_int, vp, vp, vp, vp, vp, vp,
                                       C.POINTER(_PoCsr), vp, vp]
        _port = lib
    return _port


def po_csr(a: Csr) -> _PoCsr:
    return _PoCsr(a.n, a.row_ptr.ctypes.data, a.cols.ctypes.data, a.vals.ctypes.data)


def po_layout(scheme, strategy, k, n_faces, n_elements, dim=2) -> PoLayout:
    lib = port_lib()
    lay = PoLayout()
    make = lib.po_make_layout3 if dim == 3 else lib.po_make_layout
    if make(scheme, strategy, k, n_faces, n_elements, C.byref(lay)):
        raise ValueError(lib.po_last_error().decode())
    return lay


def bsr_to_csr_pattern(brow_ptr, bcols, bs):
    """CSR pattern of a dense-block face pattern: row f*bs + r holds the
    columns g*bs + c of every block column g of block row f, ascending."""
    nb = len(brow_ptr) - 1
    cnt = np.diff(brow_ptr) * bs
    rp = np.zeros(nb * bs + 1, np.int64)
    rp[1:] = np.cumsum(np.repeat(cnt, bs))
    cols = np.empty(int(rp[-1]), np.int32)
    for f in range(nb):
        blk = (np.asarray(bcols[brow_ptr[f]:brow_ptr[f + 1]], np.int64)[:, None] * bs
               + np.arange(bs)[None, :]).ravel().astype(np.int32)
        for r in range(bs):
            i = f * bs + r
            cols[rp[i]:rp[i + 1]] = blk
    return rp, cols


def port_condense_assemble(mats, rhs, n, elim, kept, layout: PoLayout, row_ptr, cols):
    """po_condense_assemble: element condensation + element-order scatter
    into the given structural pattern (assemble.hpp:136-172)."""
    lib = port_lib()
    nelem = len(rhs) // n
    mats = np.ascontiguousarray(mats, np.float64)
    rhs = np.ascontiguousarray(rhs, np.float64)
    el = np.ascontiguousarray(elim, np.int32)
    kept = np.ascontiguousarray(kept, np.int64)
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(cols, np.int32)
    vals = np.zeros(len(cl))
    b = np.zeros(len(rp) - 1)
    pat = _PoCsr(len(rp) - 1, rp.ctypes.data, cl.ctypes.data, vals.ctypes.data)
    if lib.po_condense_assemble(nelem, n, mats.ctypes.data, rhs.ctypes.data, len(el),
                                el.ctypes.data, kept.ctypes.data, C.byref(layout), C.byref(pat),
                                vals.ctypes.data, b.ctypes.data):
        raise RuntimeError(lib.po_last_error().decode())
    return Csr(rp, cl, vals), b


def port_dg_assemble(layout: PoLayout, faces, vol, vrhs, fmat, frhs):
    """po_dg_pattern + po_dg_assemble: the 3D DG operator in CSR from shared
    local terms, scattered in the reference's order (assemble.hpp:177-346).
    faces: the Mesh3.faces() table (left, right in columns 4, 5)."""
    lib = port_lib()
    left = np.ascontiguousarray(faces[:, 4], np.int32)
    right = np.ascontiguousarray(faces[:, 5], np.int32)
    nf = len(left)
    nnz = lib.po_dg_pattern(C.byref(layout), nf, left.ctypes.data, right.ctypes.data, None, None)
    if nnz < 0:
        raise ValueError(lib.po_last_error().decode())
    n = lib.po_layout_dim(C.byref(layout))
    rp = np.zeros(n + 1, np.int64)
    cl = np.zeros(nnz, np.int32)
    lib.po_dg_pattern(C.byref(layout), nf, left.ctypes.data, right.ctypes.data, rp.ctypes.data,
                      cl.ctypes.data)
    vals = np.zeros(nnz)
    b = np.zeros(n)
    pat = _PoCsr(n, rp.ctypes.data, cl.ctypes.data, vals.ctypes.data)
    arrs = [np.ascontiguousarray(a, np.float64) for a in (vol, vrhs, fmat, frhs)]
    if lib.po_dg_assemble(C.byref(layout), nf, left.ctypes.data, right.ctypes.data,
                          *(a.ctypes.data for a in arrs), C.byref(pat), vals.ctypes.data,
                          b.ctypes.data):
        raise RuntimeError(lib.po_last_error().decode())
    return Csr(rp, cl, vals), b


def dgb_to_csr_values(row_ptr, brow_ptr, bcols, dvals, ne):
    """CSR values (the DG component-aware pattern) of DG block storage:
    velocity panel c of a block = ne x 2ne [u_c | p] columns, pressure panel
    ne x 4ne, column-major (csrc/dgb.cu). Test helper."""
    nb = len(brow_ptr) - 1
    eb = 4 * ne
    bsz = 10 * ne * ne
    out = np.empty(int(row_ptr[-1]))
    dv = np.asarray(dvals, np.float64)
    for e in range(nb):
        q0, q1 = int(brow_ptr[e]), int(brow_ptr[e + 1])
        blk = dv[q0 * bsz:q1 * bsz].reshape(q1 - q0, bsz)
        for r in range(eb):
            row = e * eb + r
            p = int(row_ptr[row])
            c, i = divmod(r, ne)
            if c < 3:
                panel = blk[:, c * 2 * ne * ne:(c + 1) * 2 * ne * ne].reshape(q1 - q0, 2 * ne, ne)
                seg = panel[:, :, i]  # (blocks, 2ne)
            else:
                panel = blk[:, 6 * ne * ne:].reshape(q1 - q0, 4 * ne, ne)
                seg = panel[:, :, i]
            out[p:p + seg.size] = seg.ravel()
    return out


class PortBlockJacobi:
    """Block-Jacobi over the entity blocks of a layout (restatement)."""

    def __init__(self, a: Csr, layout: PoLayout):
        self.lib = port_lib()
        self.layout = layout
        c = po_csr(a)
        self.inv = np.zeros(self.lib.po_bj_size(C.byref(layout)))
        bad = C.c_int64(-1)
        if self.lib.po_bj_factor(C.byref(c), C.byref(layout), self.inv, C.byref(bad)):
            raise RuntimeError(f"{self.lib.po_last_error().decode()} (block {bad.value})")
        self.n = a.n

    def apply(self, x):
        y = np.zeros(self.n)
        self.lib.po_bj_apply(C.byref(self.layout), self.inv, np.ascontiguousarray(x, np.float64), y)
        return y


class PortHierarchy:
    def __init__(self, a: Csr, layout: PoLayout, degrees, smoother_iters=2, coarse_rtol=1e-3,
                 coarse_maxit=400, smoother=0):
        self.lib = port_lib()
        self.a = a
        self._c = po_csr(a)
        deg = np.asarray(degrees, np.int32)
        self.h = self.lib.po_hier_create_ex(C.byref(self._c), C.byref(layout), deg, len(deg),
                                            smoother_iters, coarse_rtol, coarse_maxit, smoother)
        if not self.h:
            raise RuntimeError(self.lib.po_last_error().decode())
        self.nlev = len(deg)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.po_hier_destroy(self.h)

    def level_csr(self, l):
        n = self.lib.po_hier_level_dim(self.h, l)
        nnz = self.lib.po_hier_level_nnz(self.h, l)
        rp, cols, vals = np.zeros(n + 1, np.int64), np.zeros(nnz, np.int32), np.zeros(nnz)
        self.lib.po_hier_level_csr(self.h, l, rp, cols, vals)
        return Csr(rp, cols, vals)

    def level_ilu(self, l):
        lu = np.zeros(self.lib.po_hier_level_nnz(self.h, l))
        self.lib.po_hier_level_ilu(self.h, l, lu)
        return lu

    def vcycle(self, l, d):
        d = np.ascontiguousarray(d, np.float64)
        c = np.zeros(self.lib.po_hier_level_dim(self.h, l))
        self.lib.po_vcycle(self.h, l, d, c)
        return c

    def solve(self, rhs, rtol=1e-13, maxit=1000, restart=0):
        x = np.zeros(self.a.n)
        hist = np.zeros(maxit + 1)
        its, cits, vcs, rel, conv = C.c_int(), C.c_longlong(), C.c_int(), C.c_double(), C.c_int()
        self.lib.po_solve(self.h, np.ascontiguousarray(rhs, np.float64), rtol, maxit, restart, x,
                          hist.ctypes.data, C.byref(its), C.byref(cits), C.byref(vcs),
                          C.byref(rel), C.byref(conv))
        return dict(x=x, hist=hist[: its.value].copy(), its=its.value, coarse_its=cits.value,
                    vcycles=vcs.value, rel=rel.value, converged=bool(conv.value))


WIRE = os.path.join(ROOT, "oracle", "_ref", "wire_ref")
_KIND = {"family": 0, "unit-quad": 1, "unit-tri": 2}


def _wire(*args):
    import subprocess
    r = subprocess.run([WIRE, *[str(a) for a in args]], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr.strip())
    return r.stdout


def ref_write_mesh(path, kind="family", family="trapz", n=2, jitter=0.0, side="right"):
    """The reference's write_mesh of the mesh RefSystem would build."""
    _wire("mesh", _KIND[kind], family, n, jitter, SIDES[side], path)


def ref_write_matrix_market(path, kind="family", family="trapz", n=2, jitter=0.0, side="right",
                            scheme="hho-dp", strategy="v-cond", k=1):
    """The reference's write_matrix_market of the operator assembled with the
    exp manufactured data (the pattern and values of RefSystem(data='exp'))."""
    _wire("mtx", _KIND[kind], family, n, jitter, SIDES[side], SCHEMES[scheme],
          STRATEGIES[strategy], k, path)


def ref_mesh_roundtrip(src: str, dst: str):
    """The reference's read_mesh then write_mesh; returns (nv, ne, nf)."""
    return tuple(int(v) for v in _wire("roundtrip", src, dst).split())
