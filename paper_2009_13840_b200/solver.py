"""Python mirror of the reference's solver-path API, backed by the sm_100a
library (include/pstokes_cuda.h). Names and argument meaning follow
/root/reference/proj/include/pstokes (cited per class); errors map to the
reference's exception types (ValueError for std::invalid_argument,
NativeError/RuntimeError for std::runtime_error)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

SCHEMES = {"hho-dp": 0, "hho-hp": 1, "dg": 2}
STRATEGIES = {"uncond": 0, "v-cond": 1, "vp-cond": 2, "v&p-cond": 2}
SMOOTHERS = {"ilu0": 0, "bjacobi": 1}
COARSE = {"lu": 0, "gmres-ilu": 1}


class Context:
    """One CUDA context/stream (pscu_create)."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        h = C.c_void_p()
        N.check(self.lib.pscu_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.pscu_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def launches(self) -> int:
        return int(self.lib.pscu_launch_count(self.h))

    def synchronize(self):
        N.check(self.lib.pscu_synchronize(self.h))

    def timer_start(self):
        """CUDA event on the context stream (after a stream synchronize)."""
        N.check(self.lib.pscu_timer_start(self.h))

    def timer_stop(self) -> float:
        """Milliseconds since timer_start on the device timeline."""
        ms = C.c_double()
        N.check(self.lib.pscu_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def profile(self, enable: bool = True):
        N.check(self.lib.pscu_profile(self.h, int(enable)))

    PROFILE_CLASSES = {"ilu0_apply": 0, "spmv": 1, "mgs_step": 2, "other": 3, "bjacobi_apply": 4}

    def profile_read(self) -> dict:
        """{class: (launch groups, total ms, algorithmic bytes)} from CUDA
        events recorded around every launch on the context stream."""
        out = {}
        for name, k in self.PROFILE_CLASSES.items():
            cnt, ms, b = C.c_longlong(), C.c_double(), C.c_double()
            N.check(self.lib.pscu_profile_read(self.h, k, C.byref(cnt), C.byref(ms), C.byref(b)))
            out[name] = (cnt.value, ms.value, b.value)
        return out


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class CsrMatrix:
    """Device CsrMatrix (csr.hpp:19-115)."""

    def __init__(self, row_ptr, cols, vals, ctx: Context | None = None, _handle=None, _owner=None):
        self.ctx = ctx or default_context()
        self.lib = self.ctx.lib
        self._owner = _owner
        if _handle is not None:
            self.h = C.c_void_p(_handle)
            self._owned = False
        else:
            rp = np.ascontiguousarray(row_ptr, np.int64)
            cl = np.ascontiguousarray(cols, np.int32)
            vl = _f64(vals)
            h = C.c_void_p()
            N.check(self.lib.pscu_mat_create(self.ctx.h, len(rp) - 1, rp.ctypes.data,
                                             cl.ctypes.data, vl.ctypes.data, N.PSCU_HOST,
                                             C.byref(h)))
            self.h = h
            self._owned = True
        n, nnz = C.c_int64(), C.c_int64()
        self.lib.pscu_mat_dims(self.h, C.byref(n), C.byref(nnz))
        self.n, self.nnz = n.value, nnz.value

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "h", None):
            self.lib.pscu_mat_destroy(self.h)
            self.h = None

    def download(self):
        rp = np.zeros(self.n + 1, np.int64)
        cl = np.zeros(self.nnz, np.int32)
        vl = np.zeros(self.nnz)
        N.check(self.lib.pscu_mat_download(self.ctx.h, self.h, rp.ctypes.data, cl.ctypes.data,
                                           vl.ctypes.data))
        return rp, cl, vl

    @property
    def dg_modes(self) -> int:
        """0 unless DG block storage, else its modes per component."""
        return int(self.lib.pscu_mat_dg_modes(self.h))

    @property
    def block_size(self) -> int:
        """0 for CSR storage, else the dense face-block size."""
        return int(self.lib.pscu_mat_block_size(self.h))

    def download_blocks(self, vals_out=None):
        """(brow_ptr, bcols, vals) of a block-stored operator, vals column-major
        per block (into vals_out when given, e.g. a pinned buffer)."""
        bs = self.block_size
        if not bs:
            raise ValueError("not a block-stored operator")
        nb = self.n // bs
        rp = np.zeros(nb + 1, np.int64)
        N.check(self.lib.pscu_bsr_download(self.ctx.h, self.h, rp.ctypes.data, None, None))
        cl = np.zeros(int(rp[-1]), np.int32)
        vl = np.zeros(self.nnz) if vals_out is None else vals_out
        N.check(self.lib.pscu_bsr_download(self.ctx.h, self.h, None, cl.ctypes.data,
                                           vl.ctypes.data))
        return rp, cl, vl

    def multiply(self, x) -> np.ndarray:
        """CsrMatrix::multiply (csr.hpp:68-79)."""
        x = _f64(x)
        y = np.zeros(self.n)
        N.check(self.lib.pscu_spmv(self.ctx.h, self.h, x.ctypes.data, y.ctypes.data, N.PSCU_HOST))
        return y


class Ilu0:
    """Ilu0 (ilu0.hpp:17-79): factorisation and application on the device."""

    def __init__(self, a: CsrMatrix, _handle=None):
        self.a = a
        self.ctx = a.ctx
        self.lib = a.lib
        if _handle is not None:
            self.h = C.c_void_p(_handle)
            self._owned = False
        else:
            h = C.c_void_p()
            N.check(self.lib.pscu_ilu0_create(self.ctx.h, a.h, C.byref(h)))
            self.h = h
            self._owned = True

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "h", None):
            self.lib.pscu_ilu0_destroy(self.h)
            self.h = None

    def factors(self) -> np.ndarray:
        lu = np.zeros(self.a.nnz)
        N.check(self.lib.pscu_ilu0_factors(self.ctx.h, self.h, lu.ctypes.data))
        return lu

    def apply(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.zeros(self.a.n)
        N.check(self.lib.pscu_ilu0_apply(self.ctx.h, self.h, x.ctypes.data, y.ctypes.data,
                                         N.PSCU_HOST))
        return y


class BlockJacobi:
    """Block-Jacobi over the layout's entity blocks (BASELINE.json's smoother,
    a labelled alternative to the reference's Ilu0: plevels.hpp:174)."""

    def __init__(self, a: CsrMatrix, layout: N.Layout):
        self.a = a
        self.ctx = a.ctx
        self.lib = a.lib
        h = C.c_void_p()
        N.check(self.lib.pscu_bj_create(self.ctx.h, a.h, C.byref(layout), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pscu_bj_destroy(self.h)
            self.h = None

    def apply(self, x) -> np.ndarray:
        x = _f64(x)
        y = np.zeros(self.a.n)
        N.check(self.lib.pscu_bj_apply(self.ctx.h, self.h, x.ctypes.data, y.ctypes.data,
                                       N.PSCU_HOST))
        return y


@dataclass
class KrylovResult:
    """KrylovResult (gmres.hpp:29-34)."""
    x: np.ndarray
    iterations: int
    rel_residual: float
    converged: bool


def gmres(a: CsrMatrix, precond: Ilu0 | None, rhs, x0, max_it: int, rtol: float,
          side: str = "right") -> KrylovResult:
    """gmres (gmres.hpp:103-139) with A and an ILU(0) preconditioner on the
    device. ``x0=None`` means the zero vector."""
    rhs = _f64(rhs)
    x0a = None if x0 is None else _f64(x0)
    x = np.zeros(a.n)
    its, rel, conv = C.c_int(), C.c_double(), C.c_int()
    N.check(a.lib.pscu_gmres(a.ctx.h, a.h, precond.h if precond else None, rhs.ctypes.data,
                             None if x0a is None else x0a.ctypes.data, max_it, rtol,
                             1 if side == "left" else 0, x.ctypes.data, C.byref(its),
                             C.byref(rel), C.byref(conv), N.PSCU_HOST))
    return KrylovResult(x, its.value, rel.value, bool(conv.value))


def fgmres(a: CsrMatrix, precond: Ilu0 | None, rhs, max_it: int, rtol: float) -> KrylovResult:
    """fgmres (gmres.hpp:145-173) with a fixed ILU(0) (or identity)."""
    rhs = _f64(rhs)
    x = np.zeros(a.n)
    its, rel, conv = C.c_int(), C.c_double(), C.c_int()
    N.check(a.lib.pscu_fgmres(a.ctx.h, a.h, precond.h if precond else None, rhs.ctypes.data,
                              max_it, rtol, x.ctypes.data, C.byref(its), C.byref(rel),
                              C.byref(conv), N.PSCU_HOST))
    return KrylovResult(x, its.value, rel.value, bool(conv.value))


def make_layout(scheme: str | int, strategy: str | int, k: int, n_faces: int,
                n_elements: int) -> N.Layout:
    """make_layout (dof_layout.hpp:87-126) from mesh counts."""
    s = SCHEMES[scheme] if isinstance(scheme, str) else scheme
    t = STRATEGIES[strategy] if isinstance(strategy, str) else strategy
    lay = N.Layout()
    N.check(N.load().pscu_layout_make(s, t, k, n_faces, n_elements, C.byref(lay)))
    return lay


def make_layout3(k: int, n_faces: int, n_elements: int, scheme: str | int = "hho-hp",
                 strategy: str | int = "vp-cond") -> N.Layout:
    """The 3D generalisation of make_layout (BASELINE.json configs 3/5; the
    reference is 2D only): hho-hp vp-cond face blocks [vx | vy | vz | p]."""
    s = SCHEMES[scheme] if isinstance(scheme, str) else scheme
    t = STRATEGIES[strategy] if isinstance(strategy, str) else strategy
    lay = N.Layout()
    N.check(N.load().pscu_layout_make3(s, t, k, n_faces, n_elements, C.byref(lay)))
    return lay


def bsr_matrix(brow_ptr, bcols, vals, bs: int, ctx: Context | None = None) -> "CsrMatrix":
    """A CsrMatrix held in dense face-block storage (pscu_bsr_create): block
    row f covers rows [f bs, (f+1) bs), vals are the blocks column-major."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(brow_ptr, np.int64)
    cl = np.ascontiguousarray(bcols, np.int32)
    vl = _f64(vals)
    h = C.c_void_p()
    N.check(ctx.lib.pscu_bsr_create(ctx.h, len(rp) - 1, bs, rp.ctypes.data, cl.ctypes.data,
                                    vl.ctypes.data, N.PSCU_HOST, C.byref(h)))
    m = CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    m._owned = True
    return m


def dgb_matrix(brow_ptr, bcols, vals, nm: int, ctx: Context | None = None) -> "CsrMatrix":
    """A CsrMatrix in DG block storage (pscu_dgb_create; 3D DG, config 4):
    element blocks of 4 nm rows, each holding its 10 nm^2 structural entries
    as panels (velocity component c: nm x 2nm [u_c | p]; pressure: nm x 4nm).
    vals None = zero operator."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(brow_ptr, np.int64)
    cl = np.ascontiguousarray(bcols, np.int32)
    vl = None if vals is None else _f64(vals)
    h = C.c_void_p()
    N.check(ctx.lib.pscu_dgb_create(ctx.h, len(rp) - 1, nm, rp.ctypes.data, cl.ctypes.data,
                                    N.ptr(vl), N.PSCU_HOST, C.byref(h)))
    m = CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    m._owned = True
    return m


def set_values(m: "CsrMatrix", offset: int, vals, mem: int = N.PSCU_HOST, count: int = -1):
    """pscu_mat_set_values: writes vals at offset of the operator's values."""
    if mem == N.PSCU_HOST:
        v = _f64(vals)
        N.check(m.lib.pscu_mat_set_values(m.ctx.h, m.h, offset, v.size, v.ctypes.data, mem))
    else:
        N.check(m.lib.pscu_mat_set_values(m.ctx.h, m.h, offset, count, vals, mem))


def solve_system_dgb(brow_ptr, bcols, vals, nm: int, rhs, layout: N.Layout, cfg: LevelConfig,
                     ctx: Context | None = None):
    """solve_system through the one-call C ABI entry for a DG block-stored
    operator (pscu_solve_system_dgb): host buffers in, x out, all timed."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(brow_ptr, np.int64)
    cl = np.ascontiguousarray(bcols, np.int32)
    vl = _f64(vals)
    b = _f64(rhs)
    deg = np.ascontiguousarray(cfg.degrees, np.int32)
    x = np.zeros(len(b))
    hist = np.zeros(cfg.outer_maxit + 1)
    rep = N.Report()
    ncfg = cfg.native()
    N.check(ctx.lib.pscu_solve_system_dgb(ctx.h, len(rp) - 1, nm, rp.ctypes.data, cl.ctypes.data,
                                          vl.ctypes.data, b.ctypes.data, C.byref(layout),
                                          deg.ctypes.data, len(deg), C.byref(ncfg),
                                          cfg.outer_rtol, cfg.outer_maxit, cfg.restart,
                                          x.ctypes.data, hist.ctypes.data, C.byref(rep)))
    r = SolverReport(rep.outer_its, rep.coarse_its, rep.vcycles, rep.rel_residual,
                     bool(rep.converged), rep.t_setup, rep.t_solve)
    return x, hist[: rep.outer_its].copy(), r


def csr_to_bsr_values(row_ptr, cols, vals, brow_ptr, bcols, bs: int) -> np.ndarray:
    """Column-major block values of a CSR matrix whose pattern is the dense
    expansion of (brow_ptr, bcols) (e.g. an oracle-assembled operator)."""
    rp = np.asarray(row_ptr, np.int64)
    nb = len(brow_ptr) - 1
    out = np.empty(int(brow_ptr[-1]) * bs * bs)
    v = np.asarray(vals, np.float64)
    for f in range(nb):
        q0, q1 = int(brow_ptr[f]), int(brow_ptr[f + 1])
        rows = v[rp[f * bs]:rp[(f + 1) * bs]].reshape(bs, q1 - q0, bs)  # (r, block, c)
        out[q0 * bs * bs:q1 * bs * bs] = np.transpose(rows, (1, 2, 0)).ravel()
    return out


def layout_dim(lay: N.Layout) -> int:
    return int(N.load().pscu_layout_dim(C.byref(lay)))


def coarse_to_fine_map(fine: N.Layout, coarse: N.Layout) -> np.ndarray:
    """coarse_to_fine_map (plevels.hpp:47-72)."""
    m = np.zeros(layout_dim(coarse), np.int64)
    N.check(N.load().pscu_coarse_to_fine(C.byref(fine), C.byref(coarse), m.ctypes.data))
    return m


def inherit_matrix(fine: CsrMatrix, lf: N.Layout, lc: N.Layout) -> CsrMatrix:
    """inherit_matrix (plevels.hpp:93-113) as a device gather."""
    h = C.c_void_p()
    N.check(fine.lib.pscu_inherit(fine.ctx.h, fine.h, C.byref(lf), C.byref(lc), C.byref(h)))
    m = CsrMatrix(None, None, None, ctx=fine.ctx, _handle=h.value)
    m._owned = True
    return m


@dataclass
class LevelConfig:
    """LevelConfig (plevels.hpp:23-42) + smoother kind and FGMRES restart."""
    degrees: list
    smoother_iters: int = 2
    coarse: str = "lu"
    coarse_rtol: float = 1e-3
    coarse_maxit: int = 400
    outer_rtol: float = 1e-13
    outer_maxit: int = 1000
    smoother: str = "ilu0"
    restart: int = 0

    def native(self) -> N.LevelCfg:
        return N.LevelCfg(SMOOTHERS[self.smoother], self.smoother_iters, COARSE[self.coarse],
                          self.coarse_rtol, self.coarse_maxit)


@dataclass
class SolverReport:
    """SolverReport (gmres.hpp:19-27)."""
    outer_its: int
    coarse_its: int
    vcycles: int
    rel_residual: float
    converged: bool
    t_setup: float
    t_solve: float


class LevelHierarchy:
    """LevelHierarchy (plevels.hpp:125-212) on the device."""

    def __init__(self, a: CsrMatrix, layout: N.Layout, cfg: LevelConfig):
        self.a = a
        self.cfg = cfg
        self.lib = a.lib
        self.ctx = a.ctx
        deg = np.ascontiguousarray(cfg.degrees, np.int32)
        self._deg = deg
        h = C.c_void_p()
        ncfg = cfg.native()
        N.check(self.lib.pscu_hier_create(self.ctx.h, a.h, C.byref(layout), deg.ctypes.data,
                                          len(deg), C.byref(ncfg), C.byref(h)))
        self.h = h
        self.nlev = len(deg)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.pscu_hier_destroy(self.h)
            self.h = None

    def level_matrix(self, l: int) -> CsrMatrix:
        p = self.lib.pscu_hier_level_mat(self.h, l)
        return CsrMatrix(None, None, None, ctx=self.ctx, _handle=p, _owner=self)

    def level_ilu(self, l: int) -> Ilu0:
        p = self.lib.pscu_hier_level_ilu(self.h, l)
        if not p:
            raise ValueError("level has no ILU(0) factor")
        return Ilu0(self.level_matrix(l), _handle=p)

    def vcycle(self, l: int, defect) -> np.ndarray:
        d = _f64(defect)
        c = np.zeros_like(d)
        N.check(self.lib.pscu_vcycle(self.ctx.h, self.h, l, d.ctypes.data, c.ctypes.data,
                                     N.PSCU_HOST))
        return c

    def coarse_iterations(self) -> int:
        return int(self.lib.pscu_hier_coarse_its(self.h))

    def reset_counters(self):
        self.lib.pscu_hier_reset(self.h)

    def solve(self, rhs, rtol: float | None = None, maxit: int | None = None,
              restart: int | None = None, history: bool = True):
        """fgmres(A, vcycle) (plevels.hpp:217-239) -> (x, hist, SolverReport)."""
        rhs = _f64(rhs)
        rtol = self.cfg.outer_rtol if rtol is None else rtol
        maxit = self.cfg.outer_maxit if maxit is None else maxit
        restart = self.cfg.restart if restart is None else restart
        x = np.zeros(self.a.n)
        hist = np.zeros(maxit + 1)
        rep = N.Report()
        N.check(self.lib.pscu_solve(self.ctx.h, self.h, rhs.ctypes.data, rtol, maxit, restart,
                                    x.ctypes.data, hist.ctypes.data if history else None,
                                    C.byref(rep), N.PSCU_HOST))
        r = SolverReport(rep.outer_its, rep.coarse_its, rep.vcycles, rep.rel_residual,
                         bool(rep.converged), rep.t_setup, rep.t_solve)
        return x, hist[: rep.outer_its].copy(), r


def solve_system(row_ptr, cols, vals, rhs, layout: N.Layout, cfg: LevelConfig,
                 ctx: Context | None = None):
    """solve_system (plevels.hpp:217-239) through the one-call C ABI entry:
    host CSR + rhs in, x out; upload, setup and solve are all inside the
    timed t_solve. Returns (x, hist, SolverReport)."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(cols, np.int32)
    vl = _f64(vals)
    b = _f64(rhs)
    deg = np.ascontiguousarray(cfg.degrees, np.int32)
    n = len(rp) - 1
    x = np.zeros(n)
    hist = np.zeros(cfg.outer_maxit + 1)
    rep = N.Report()
    ncfg = cfg.native()
    N.check(ctx.lib.pscu_solve_system(ctx.h, n, rp.ctypes.data, cl.ctypes.data, vl.ctypes.data,
                                      b.ctypes.data, C.byref(layout), deg.ctypes.data, len(deg),
                                      C.byref(ncfg), cfg.outer_rtol, cfg.outer_maxit, cfg.restart,
                                      x.ctypes.data, hist.ctypes.data, C.byref(rep)))
    r = SolverReport(rep.outer_its, rep.coarse_its, rep.vcycles, rep.rel_residual,
                     bool(rep.converged), rep.t_setup, rep.t_solve)
    return x, hist[: rep.outer_its].copy(), r


def solve_system_bsr(brow_ptr, bcols, vals, bs: int, rhs, layout: N.Layout, cfg: LevelConfig,
                     ctx: Context | None = None):
    """solve_system through the one-call C ABI entry for a face-block
    operator (pscu_solve_system_bsr): host buffers in, x out, everything
    inside the timed t_solve. Returns (x, hist, SolverReport)."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(brow_ptr, np.int64)
    cl = np.ascontiguousarray(bcols, np.int32)
    vl = _f64(vals)
    b = _f64(rhs)
    deg = np.ascontiguousarray(cfg.degrees, np.int32)
    x = np.zeros(len(b))
    hist = np.zeros(cfg.outer_maxit + 1)
    rep = N.Report()
    ncfg = cfg.native()
    N.check(ctx.lib.pscu_solve_system_bsr(ctx.h, len(rp) - 1, bs, rp.ctypes.data, cl.ctypes.data,
                                          vl.ctypes.data, b.ctypes.data, C.byref(layout),
                                          deg.ctypes.data, len(deg), C.byref(ncfg),
                                          cfg.outer_rtol, cfg.outer_maxit, cfg.restart,
                                          x.ctypes.data, hist.ctypes.data, C.byref(rep)))
    r = SolverReport(rep.outer_its, rep.coarse_its, rep.vcycles, rep.rel_residual,
                     bool(rep.converged), rep.t_setup, rep.t_solve)
    return x, hist[: rep.outer_its].copy(), r


def condense_elements(mats, rhs, elim, ctx: Context | None = None):
    """Batched condense_element (condense.hpp:57-97) over elements sharing one
    local size and elimination list. mats: (nelem, n, n), rhs: (nelem, n).
    Returns dict(schur, reduced_rhs, elim_coupling, elim_rhs) as arrays of
    per-element matrices (row-major numpy views of column-major blocks)."""
    ctx = ctx or default_context()
    mats = np.asarray(mats, np.float64)
    nelem, n, _ = mats.shape
    colmajor = np.ascontiguousarray(np.transpose(mats, (0, 2, 1)))
    b = _f64(rhs).reshape(nelem, n)
    el = np.ascontiguousarray(elim, np.int32)
    ne = len(el)
    nk = n - ne
    schur = np.zeros((nelem, nk, nk))
    rr = np.zeros((nelem, nk))
    coup = np.zeros((nelem, max(ne, 1) * nk))
    er = np.zeros((nelem, max(ne, 1)))
    bad = C.c_int(-1)
    N.check(ctx.lib.pscu_condense_batch(ctx.h, nelem, n, colmajor.ctypes.data, b.ctypes.data, ne,
                                        el.ctypes.data, schur.ctypes.data, rr.ctypes.data,
                                        coup.ctypes.data, er.ctypes.data, C.byref(bad),
                                        N.PSCU_HOST))
    return dict(schur=np.transpose(schur, (0, 2, 1)), reduced_rhs=rr,
                elim_coupling=np.transpose(coup[:, : ne * nk].reshape(nelem, nk, ne), (0, 2, 1)),
                elim_rhs=er[:, :ne])


def recover_elements(elim, kept_global, elim_coupling, elim_rhs, x, ctx: Context | None = None):
    """ElementCondensation::recover (condense.hpp:28-38) for a batch of
    elements sharing one local size and elimination list, i.e.
    StokesSystem::recover_solution (assemble.hpp:58-66) on the device.
    kept_global: (nelem, nk) retained global ids; elim_coupling: (nelem, ne,
    nk); elim_rhs: (nelem, ne); x: the global solution. Returns the full local
    vectors (nelem, n) in local dof order."""
    ctx = ctx or default_context()
    el = np.ascontiguousarray(elim, np.int32)
    kept = np.ascontiguousarray(kept_global, np.int64)
    nelem, nk = kept.shape
    ne = len(el)
    n = nk + ne
    coup = np.ascontiguousarray(np.transpose(np.asarray(elim_coupling, np.float64).reshape(
        nelem, ne, nk), (0, 2, 1)))  # column-major blocks
    er = _f64(np.asarray(elim_rhs, np.float64).reshape(nelem, ne))
    xx = _f64(x)
    locals_ = np.zeros((nelem, n))
    N.check(ctx.lib.pscu_recover_batch(ctx.h, nelem, n, ne, el.ctypes.data, kept.ctypes.data,
                                       coup.ctypes.data, er.ctypes.data, xx.ctypes.data,
                                       locals_.ctypes.data, N.PSCU_HOST))
    return locals_
