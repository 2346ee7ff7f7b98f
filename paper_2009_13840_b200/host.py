"""ctypes binding of the host input producer (include/pstokes_host.h) and
the assemble_stokes pipeline: host local blocks -> device condensation and
assembly (pscu_condense_assemble)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .build import HOST_LIB

SIDES = {"left": 0, "right": 1, "top": 2, "bottom": 3}
DATA = {"zero": 0, "exp": 1, "sincos": 2}
SCHEMES = {"hho-dp": 0, "hho-hp": 1}
STRATEGIES = {"uncond": 0, "v-cond": 1, "vp-cond": 2, "v&p-cond": 2}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"host producer library missing: {HOST_LIB}")
        lib = C.CDLL(HOST_LIB)
        vp = C.c_void_p
        lib.psh_last_error.restype = C.c_char_p
        lib.psh_mesh_unit_square.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                             C.POINTER(vp)]
        lib.psh_mesh_family.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]
        lib.psh_mesh_destroy.argtypes = [vp]
        lib.psh_mesh_counts.argtypes = [vp, vp]
        lib.psh_mesh_faces.argtypes = [vp, vp]
        lib.psh_mesh_vertices.argtypes = [vp, vp]
        lib.psh_build.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  C.POINTER(vp)]
        lib.psh_system_destroy.argtypes = [vp]
        lib.psh_system_info.argtypes = [vp, vp]
        for f in ("psh_local_mats", "psh_local_rhs", "psh_elim", "psh_kept_global", "psh_row_ptr",
                  "psh_cols"):
            getattr(lib, f).restype = vp
            getattr(lib, f).argtypes = [vp]
        lib.psh_build_seconds.restype = C.c_double
        lib.psh_build_seconds.argtypes = [vp]
        lib.psh_mesh_write.argtypes = [vp, C.c_char_p]
        lib.psh_mesh_read.argtypes = [C.c_char_p, C.POINTER(vp)]
        lib.psh_write_matrix_market.argtypes = [C.c_int64, vp, vp, vp, C.c_char_p]
        lib.psh_error_tables.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, vp, vp]
        _lib = lib
    return _lib


def _check(rc):
    if rc:
        msg = load().psh_last_error().decode()
        raise ValueError(msg) if rc == 1 else RuntimeError(msg)


class Mesh:
    """2D mesh (mesh.hpp) built by the host producer."""

    def __init__(self, h):
        self.lib = load()
        self.h = h
        c = np.zeros(3, np.int64)
        self.lib.psh_mesh_counts(h, c.ctypes.data)
        self.n_vertices, self.n_elements, self.n_faces = (int(v) for v in c)

    @classmethod
    def unit_square(cls, n: int, tri: bool = False, jitter: float = 0.0, seed: int = 0,
                    neumann: str = "top") -> "Mesh":
        h = C.c_void_p()
        _check(load().psh_mesh_unit_square(n, int(tri), jitter, seed, SIDES[neumann], C.byref(h)))
        return cls(h)

    @classmethod
    def family(cls, family: str, n: int, neumann: str = "right") -> "Mesh":
        h = C.c_void_p()
        _check(load().psh_mesh_family(family.encode(), n, SIDES[neumann], C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.psh_mesh_destroy(self.h)
            self.h = None

    @classmethod
    def read(cls, path: str) -> "Mesh":
        """read_mesh (mesh.hpp:562-645): pmesh2 v1 file, faces derived when nf = 0."""
        h = C.c_void_p()
        _check(load().psh_mesh_read(os.fsencode(path), C.byref(h)))
        return cls(h)

    def write(self, path: str) -> None:
        """write_mesh (mesh.hpp:540-560), byte-compatible with the reference."""
        _check(self.lib.psh_mesh_write(self.h, os.fsencode(path)))

    def faces(self) -> np.ndarray:
        f = np.zeros(5 * self.n_faces, np.int32)
        self.lib.psh_mesh_faces(self.h, f.ctypes.data)
        return f.reshape(-1, 5)

    def vertices(self) -> np.ndarray:
        v = np.zeros(2 * self.n_vertices)
        self.lib.psh_mesh_vertices(self.h, v.ctypes.data)
        return v.reshape(-1, 2)


def write_matrix_market(row_ptr, cols, vals, path: str) -> None:
    """write_matrix_market (csr.hpp:98-111): 1-based coordinate triplets at
    precision 17, byte-compatible with the reference's export."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cl = np.ascontiguousarray(cols, np.int32)
    vl = np.ascontiguousarray(vals, np.float64)
    _check(load().psh_write_matrix_market(len(rp) - 1, rp.ctypes.data, cl.ctypes.data,
                                          vl.ctypes.data, os.fsencode(path)))


def _view(ptr, dtype, count):
    if count == 0:
        return np.zeros(0, dtype)
    buf = (C.c_char * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype, count=count)


class LocalSystem:
    """Per-element local blocks, layout and pattern (assemble_hho front end)."""

    def __init__(self, mesh: Mesh, scheme: str, strategy: str, k: int, data: str = "sincos",
                 eta: float = 0.0, nthreads: int = 0):
        self.lib = load()
        self.mesh = mesh
        self.data = DATA[data]
        h = C.c_void_p()
        _check(self.lib.psh_build(mesh.h, SCHEMES[scheme], STRATEGIES[strategy], k, DATA[data],
                                  eta, nthreads, C.byref(h)))
        self.h = h
        info = np.zeros(14, np.int64)
        self.lib.psh_system_info(h, info.ctypes.data)
        (self.nelem, self.n_local, self.n_elim, self.n_keep, self.dim, self.nnz, self.scheme,
         self.strategy, self.k, self.n_faces, self.face_vel, self.face_press, self.elem_vel,
         self.elem_press) = (int(v) for v in info)
        self.seconds = self.lib.psh_build_seconds(h)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.psh_system_destroy(self.h)
            self.h = None

    def layout(self) -> N.Layout:
        return N.Layout(self.scheme, self.strategy, self.k, self.n_faces, self.nelem,
                        self.face_vel, self.face_press, self.elem_vel, self.elem_press)

    def mats(self):
        n = self.n_local
        return _view(self.lib.psh_local_mats(self.h), np.float64, self.nelem * n * n)

    def rhs(self):
        return _view(self.lib.psh_local_rhs(self.h), np.float64, self.nelem * self.n_local)

    def elim(self):
        return _view(self.lib.psh_elim(self.h), np.int32, self.n_elim)

    def kept_global(self):
        return _view(self.lib.psh_kept_global(self.h), np.int64, self.nelem * self.n_keep)

    def row_ptr(self):
        return _view(self.lib.psh_row_ptr(self.h), np.int64, self.dim + 1)

    def cols(self):
        return _view(self.lib.psh_cols(self.h), np.int32, self.nnz)


@dataclass
class Recovery:
    """Per-element recovery data of the static condensation
    (ElementCondensation, condense.hpp:28-38): elim_coupling (nelem, ne, nk),
    elim_rhs (nelem, ne), the eliminated local dofs and the retained global ids."""
    elim: np.ndarray
    kept_global: np.ndarray
    elim_coupling: np.ndarray
    elim_rhs: np.ndarray


def assemble_stokes(local: LocalSystem, ctx=None, recovery: bool = False):
    """assemble_stokes (assemble.hpp:348-353) for the HHO schemes: device
    condensation + assembly of the host-built local blocks. Returns the
    condensed operator as a device CsrMatrix and the reduced rhs (and the
    Recovery data when asked, for recover_solution / error_norms)."""
    from . import solver as S

    ctx = ctx or S.default_context()
    h = C.c_void_p()
    rhs = np.zeros(local.dim)
    lay = local.layout()
    ne, nk = local.n_elim, local.n_keep
    coup = np.zeros(local.nelem * ne * nk) if recovery else None
    erhs = np.zeros(local.nelem * ne) if recovery else None
    N.check(ctx.lib.pscu_condense_assemble(
        ctx.h, local.nelem, local.n_local, local.lib.psh_local_mats(local.h),
        local.lib.psh_local_rhs(local.h), local.n_elim, local.lib.psh_elim(local.h),
        local.lib.psh_kept_global(local.h), local.dim, local.lib.psh_row_ptr(local.h),
        local.lib.psh_cols(local.h), C.byref(lay), N.PSCU_HOST, C.byref(h), rhs.ctypes.data,
        coup.ctypes.data if recovery else None, erhs.ctypes.data if recovery else None))
    m = S.CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    m._owned = True
    if not recovery:
        return m, rhs
    # column-major (ne x nk) blocks -> (nelem, ne, nk)
    rec = Recovery(local.elim().copy(), local.kept_global().reshape(local.nelem, nk).copy(),
                   coup.reshape(local.nelem, nk, ne).transpose(0, 2, 1), erhs.reshape(local.nelem, ne))
    return m, rhs, rec


@dataclass
class ErrorNorms:
    """ErrorNorms (errors.hpp:27-30)."""
    u: float
    grad_u: float
    p: float
    div_u: float

    def as_array(self) -> np.ndarray:
        return np.array([self.u, self.grad_u, self.p, self.div_u])


def error_tables(local: LocalSystem, e0: int = 0, nelem: int | None = None, out=None):
    """psh_error_tables: (dims, tables) of elements [e0, e0 + nelem)."""
    dims = np.zeros(11, np.int32)
    lib = local.lib
    _check(lib.psh_error_tables(local.mesh.h, local.scheme, local.k, local.data, 0, 0, 0, None,
                                dims.ctypes.data))
    if nelem is None:
        nelem = local.nelem - e0
    if out is None:
        out = np.zeros(int(nelem) * int(dims[4]))
    _check(lib.psh_error_tables(local.mesh.h, local.scheme, local.k, local.data, e0, nelem, 0,
                                out.ctypes.data, dims.ctypes.data))
    return dims, out


def error_norms(local: LocalSystem, x, rec: Recovery, batch: int = 8192, ctx=None,
                return_locals: bool = False):
    """StokesSystem::recover_solution (assemble.hpp:58-66) and error_norms
    (errors.hpp:32-117) on the device, streamed over element batches: the
    host produces each batch's point tables into a pinned buffer, the device
    recovers the batch's local vectors from x (pscu_recover_batch) and adds
    its error integrals to the running sums (pscu_error_accumulate), in the
    reference's order, so the norms are the reference's bit for bit. x: the
    global solution (host or torch CUDA tensor)."""
    import torch

    from . import solver as S

    ctx = ctx or S.default_context()
    dev = torch.device("cuda", 0)
    dims, _ = error_tables(local, 0, 0)
    per, nloc = int(dims[4]), int(dims[8])
    ne, nk = len(rec.elim), rec.kept_global.shape[1]
    if nloc != ne + nk:
        raise ValueError("error_norms: recovery data does not match the local layout")
    xd = torch.as_tensor(np.ascontiguousarray(x, np.float64), device=dev) \
        if not torch.is_tensor(x) else x.to(dev, torch.float64).contiguous()
    el = np.ascontiguousarray(rec.elim, np.int32)
    # recovery data on the device once, column-major blocks like the kernel reads
    kept = torch.as_tensor(np.ascontiguousarray(rec.kept_global, np.int64), device=dev)
    coup = torch.as_tensor(np.ascontiguousarray(np.transpose(rec.elim_coupling, (0, 2, 1))),
                           device=dev)
    erhs = torch.as_tensor(np.ascontiguousarray(rec.elim_rhs, np.float64), device=dev)
    acc = torch.zeros(4, dtype=torch.float64, device=dev)
    nb = min(batch, local.nelem)
    pin = N.PinnedArray(nb * per)
    tab = torch.empty(nb * per, dtype=torch.float64, device=dev)
    loc = torch.empty(nb * nloc, dtype=torch.float64, device=dev)
    all_locals = torch.empty((local.nelem, nloc), dtype=torch.float64, device=dev) \
        if return_locals else None
    dp = dims.ctypes.data
    for e0 in range(0, local.nelem, nb):
        m = min(nb, local.nelem - e0)
        error_tables(local, e0, m, pin.a)
        tab[:m * per].copy_(torch.from_numpy(pin.a[:m * per]))
        torch.cuda.current_stream(dev).synchronize()
        N.check(ctx.lib.pscu_recover_batch(ctx.h, m, nloc, ne, el.ctypes.data,
                                           kept[e0:e0 + m].data_ptr(), coup[e0:e0 + m].data_ptr(),
                                           erhs[e0:e0 + m].data_ptr(), xd.data_ptr(),
                                           loc.data_ptr(), N.PSCU_DEVICE))
        N.check(ctx.lib.pscu_error_accumulate(ctx.h, dp, m, tab.data_ptr(), loc.data_ptr(),
                                              acc.data_ptr(), N.PSCU_DEVICE))
        if return_locals:
            all_locals[e0:e0 + m].copy_(loc[:m * nloc].view(m, nloc))
    sq = np.sqrt(acc.cpu().numpy())
    out = ErrorNorms(*(float(v) for v in sq))
    return (out, all_locals.cpu().numpy()) if return_locals else out


# ---------------------------------------------------------------------------
# 3D (BASELINE.json configs 3 and 5): hexahedral unit cube, HHO-hp vp-cond
# ---------------------------------------------------------------------------

DATA3 = {"zero": 0, "random": 3, "manufactured": 4}


def load3():
    lib = load()
    if not getattr(lib, "_psh3", False):
        vp = C.c_void_p
        lib.psh3_last_error.restype = C.c_char_p
        lib.psh_mesh_unit_cube.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int, C.POINTER(vp)]
        lib.psh_mesh3_destroy.argtypes = [vp]
        for f in ("psh_mesh3_counts", "psh_mesh3_faces", "psh_mesh3_element_faces",
                  "psh_mesh3_vertices"):
            getattr(lib, f).argtypes = [vp, vp]
        lib.psh3_hp_info.argtypes = [C.c_int, vp]
        lib.psh3_hp_elim.argtypes = [C.c_int, vp]
        lib.psh3_hp_keep_pos.argtypes = [C.c_int, vp]
        lib.psh3_local_blocks.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                          C.c_int, C.c_int, vp, vp]
        lib.psh3_block_pattern.restype = C.c_int64
        lib.psh3_block_pattern.argtypes = [vp, vp, vp]
        lib.psh3_face_projection.argtypes = [vp, C.c_int, vp]
        lib.psh3_geometry.argtypes = [vp, vp]
        lib.psh3_device_inputs.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, vp,
                                           vp, vp, vp, vp, vp]
        lib.psh3_dg_info.argtypes = [C.c_int, vp]
        lib.psh3_dg_block_pattern.restype = C.c_int64
        lib.psh3_dg_block_pattern.argtypes = [vp, vp, vp]
        lib.psh3_dg_local.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int, vp,
                                      vp, vp, vp]
        lib.psh3_dg_rows.argtypes = [vp, C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_int,
                                     C.c_int, vp, vp, C.c_int, vp, vp]
        lib.psh3_dg_l2_errors.argtypes = [vp, C.c_int, vp, vp]
        lib._psh3 = True
    return lib


def _check3(rc):
    if rc:
        msg = load3().psh3_last_error().decode()
        raise ValueError(msg) if rc == 1 else RuntimeError(msg)


class Mesh3:
    """Hexahedral unit-cube mesh (3D generalisation of mesh.hpp; see
    host/pstokes_host3d.cpp for the recipe and the non-planar-face choice)."""

    def __init__(self, n: int, jitter: float = 0.0, seed: int = 0, neumann_top: bool = True):
        self.lib = load3()
        h = C.c_void_p()
        _check3(self.lib.psh_mesh_unit_cube(n, jitter, seed, int(neumann_top), C.byref(h)))
        self.h = h
        self.n = n
        c = np.zeros(3, np.int64)
        self.lib.psh_mesh3_counts(h, c.ctypes.data)
        self.n_vertices, self.n_elements, self.n_faces = (int(v) for v in c)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.psh_mesh3_destroy(self.h)
            self.h = None

    def faces(self) -> np.ndarray:
        f = np.zeros(7 * self.n_faces, np.int32)
        self.lib.psh_mesh3_faces(self.h, f.ctypes.data)
        return f.reshape(-1, 7)

    def element_faces(self) -> np.ndarray:
        f = np.zeros(6 * self.n_elements, np.int32)
        self.lib.psh_mesh3_element_faces(self.h, f.ctypes.data)
        return f.reshape(-1, 6)

    def vertices(self) -> np.ndarray:
        v = np.zeros(3 * self.n_vertices)
        self.lib.psh_mesh3_vertices(self.h, v.ctypes.data)
        return v.reshape(-1, 3)

    def geometry(self):
        out = np.zeros(2 * self.n_elements)
        _check3(self.lib.psh3_geometry(self.h, out.ctypes.data))
        return out[: self.n_elements], out[self.n_elements:]

    def block_pattern(self):
        lib = self.lib
        nb = lib.psh3_block_pattern(self.h, None, None)
        rp = np.zeros(self.n_faces + 1, np.int64)
        cols = np.zeros(nb, np.int32)
        lib.psh3_block_pattern(self.h, rp.ctypes.data, cols.ctypes.data)
        return rp, cols

    def device_inputs(self, k: int, data: str = "random", seed: int = 0, e0: int = 0,
                      e1: int | None = None, mesh_tables: bool = True) -> dict:
        """psh3_device_inputs: what the device local-block producer reads for
        elements [e0, e1) (hex, ef, es, coef; batch-relative) and, with
        mesh_tables, the whole-mesh vertices, face table and quadrature rule."""
        e1 = self.n_elements if e1 is None else e1
        m = e1 - e0
        npk = (k + 1) * (k + 2) * (k + 3) // 6
        d = dict(hex=np.zeros(8 * m, np.int32), ef=np.zeros(6 * m, np.int32),
                 es=np.zeros(6 * m, np.int32),
                 coef=np.zeros(3 * npk * m) if DATA3[data] == 3 else None)
        gl = np.zeros(16) if mesh_tables else None
        ftab = np.zeros(5 * self.n_faces, np.int32) if mesh_tables else None
        npts = self.lib.psh3_device_inputs(self.h, k, DATA3[data], seed, e0, e1,
                                           d["hex"].ctypes.data, d["ef"].ctypes.data,
                                           d["es"].ctypes.data, N.ptr(ftab), N.ptr(gl),
                                           N.ptr(d["coef"]))
        if npts < 0:
            _check3(-npts)
        if mesh_tables:
            d.update(nq1=npts, gl=np.ascontiguousarray(gl[:2 * npts]), ftab=ftab,
                     xyz=self.vertices().ravel())
        return d

    def face_projection(self, k: int) -> np.ndarray:
        nf = (k + 1) * (k + 2) // 2
        out = np.zeros(self.n_faces * 4 * nf)
        _check3(self.lib.psh3_face_projection(self.h, k, out.ctypes.data))
        return out


class DgLocal3:
    """3D DG (BR2) at degree k (BASELINE.json config 4; the reference's DG,
    assemble.hpp:177-346, with three velocity components): element blocks
    [ux | uy | uz | p] of ne = dim P^k(3D) modes each."""

    def __init__(self, k: int):
        info = np.zeros(2, np.int32)
        _check3(load3().psh3_dg_info(k, info.ctypes.data))
        self.k = k
        self.ne, self.elem_block = int(info[0]), int(info[1])

    @staticmethod
    def block_pattern(mesh: "Mesh3"):
        lib = load3()
        nb = lib.psh3_dg_block_pattern(mesh.h, None, None)
        rp = np.zeros(mesh.n_elements + 1, np.int64)
        cols = np.zeros(nb, np.int32)
        lib.psh3_dg_block_pattern(mesh.h, rp.ctypes.data, cols.ctypes.data)
        return rp, cols

    def local_terms(self, mesh: "Mesh3", data: str = "random", seed: int = 0, eta: float = 0.0,
                    nthreads: int = 0):
        """(vol, vrhs, fmat, frhs) for the oracle's reference-order scatter."""
        nl = self.elem_block
        vol = np.zeros(mesh.n_elements * nl * nl)
        vr = np.zeros(mesh.n_elements * nl)
        fm = np.zeros(mesh.n_faces * 4 * nl * nl)
        fr = np.zeros(mesh.n_faces * 2 * nl)
        _check3(load3().psh3_dg_local(mesh.h, self.k, DATA3[data], seed, eta, nthreads,
                                      vol.ctypes.data, vr.ctypes.data, fm.ctypes.data,
                                      fr.ctypes.data))
        return vol, vr, fm, fr

    def rows(self, mesh: "Mesh3", brow_ptr, bcols, e0: int, e1: int, data: str = "random",
             seed: int = 0, eta: float = 0.0, nthreads: int = 0, out=None):
        """Block rows [e0, e1) in DG block storage (10 ne^2 per block) and
        their loads (psh3_dg_rows)."""
        rp = np.ascontiguousarray(brow_ptr, np.int64)
        cl = np.ascontiguousarray(bcols, np.int32)
        nblk = int(rp[e1] - rp[e0])
        if out is None:
            vals = np.zeros(nblk * 10 * self.ne * self.ne)
            rhs = np.zeros((e1 - e0) * self.elem_block)
        else:
            vals, rhs = out
        _check3(load3().psh3_dg_rows(mesh.h, self.k, DATA3[data], seed, eta, e0, e1,
                                     rp.ctypes.data, cl.ctypes.data, nthreads, N.ptr(vals),
                                     N.ptr(rhs)))
        return vals, rhs

    def l2_errors(self, mesh: "Mesh3", x) -> tuple:
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(2)
        _check3(load3().psh3_dg_l2_errors(mesh.h, self.k, x.ctypes.data, out.ctypes.data))
        return float(out[0]), float(out[1])


class HpLocal3:
    """HHO-hp vp-cond local structure at face degree k (3D): sizes, the
    eliminated local dofs and the face-block position of every retained dof."""

    def __init__(self, k: int):
        lib = load3()
        self.k = k
        info = np.zeros(8, np.int32)
        _check3(lib.psh3_hp_info(k, info.ctypes.data))
        (self.n_local, self.n_elim, self.n_keep, self.face_vel, self.face_press, self.face_block,
         self.nfaces, self.ne) = (int(v) for v in info)
        self.elim = np.zeros(self.n_elim, np.int32)
        _check3(lib.psh3_hp_elim(k, self.elim.ctypes.data))
        pos = np.zeros(2 * self.n_keep, np.int32)
        _check3(lib.psh3_hp_keep_pos(k, pos.ctypes.data))
        self.keep_pos = pos.reshape(-1, 2)

    def kept_global(self, element_faces: np.ndarray) -> np.ndarray:
        """Retained global ids per element (nelem x n_keep)."""
        ef = np.asarray(element_faces, np.int64)
        return ef[:, self.keep_pos[:, 0]] * self.face_block + self.keep_pos[:, 1][None, :]

    def local_blocks(self, mesh: Mesh3, e0: int, e1: int, data: str = "random", seed: int = 0,
                     eta: float = 0.0, nthreads: int = 0, out=None):
        n = self.n_local
        m = e1 - e0
        if out is None:
            mats = np.zeros(m * n * n)
            rhs = np.zeros(m * n)
        else:
            mats, rhs = out
        _check3(load3().psh3_local_blocks(mesh.h, self.k, DATA3[data], seed, eta, e0, e1, nthreads,
                                          N.ptr(mats), N.ptr(rhs)))
        return mats, rhs


def _assemble_stokes3_device(mesh, k, data, seed, eta, batch, ctx, recovery):
    """assemble_stokes3 with the local blocks built on the device: per batch
    the host packs the element connectivity (and data-3 coefficients), the
    device builds the blocks into a device buffer and condenses / scatters
    them in place (pscu_local_blocks3 + pscu_assembly_add, device memory)."""
    import time

    import torch

    from . import solver as S

    dev = torch.device("cuda", 0)
    L = HpLocal3(k)
    brp, bcols = mesh.block_pattern()
    h = C.c_void_p()
    N.check(ctx.lib.pscu_assembly_begin(ctx.h, mesh.n_faces, L.face_block, brp.ctypes.data,
                                        bcols.ctypes.data, C.byref(h)))
    A = S.CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    A._owned = True
    keep_pos = np.ascontiguousarray(L.keep_pos, np.int32)
    n = L.n_local
    nb = min(batch, mesh.n_elements)
    tab = mesh.device_inputs(k, data, seed, 0, 0)
    xyz = torch.as_tensor(tab["xyz"], device=dev)
    ftab = torch.as_tensor(tab["ftab"], device=dev)
    gl = torch.as_tensor(tab["gl"], device=dev)
    mats = torch.empty(nb * n * n, dtype=torch.float64, device=dev)
    rhs = torch.empty(nb * n, dtype=torch.float64, device=dev)
    eta_v = eta if eta > 0.0 else 3.0 * (k + 1) * (k + 1)
    coup = erhs = None
    if recovery:
        coup = np.empty((mesh.n_elements, L.n_elim, L.n_keep))
        erhs = np.empty((mesh.n_elements, L.n_elim))
        cpd = torch.empty(nb * L.n_elim * L.n_keep, dtype=torch.float64, device=dev)
        epd = torch.empty(nb * L.n_elim, dtype=torch.float64, device=dev)
    t_local = t_dev = 0.0
    for e0 in range(0, mesh.n_elements, nb):
        e1 = min(mesh.n_elements, e0 + nb)
        m = e1 - e0
        d = mesh.device_inputs(k, data, seed, e0, e1, mesh_tables=False)
        hx = torch.as_tensor(d["hex"], device=dev)
        ef = torch.as_tensor(d["ef"], device=dev)
        es = torch.as_tensor(d["es"], device=dev)
        cf = torch.as_tensor(d["coef"], device=dev) if d["coef"] is not None else None
        torch.cuda.current_stream(dev).synchronize()
        t0 = time.perf_counter()
        N.check(ctx.lib.pscu_local_blocks3(ctx.h, k, DATA3[data], eta_v, tab["nq1"], gl.data_ptr(),
                                           mesh.n_vertices, xyz.data_ptr(), mesh.n_faces,
                                           ftab.data_ptr(), m, hx.data_ptr(), ef.data_ptr(),
                                           es.data_ptr(), N.ptr(cf), mats.data_ptr(),
                                           rhs.data_ptr(), N.PSCU_DEVICE))
        t1 = time.perf_counter()
        N.check(ctx.lib.pscu_assembly_add(ctx.h, A.h, e0, m, n, mats.data_ptr(), rhs.data_ptr(),
                                          L.n_elim, L.elim.ctypes.data, ef.data_ptr(), 6,
                                          keep_pos.ctypes.data,
                                          cpd.data_ptr() if recovery else None,
                                          epd.data_ptr() if recovery else None, N.PSCU_DEVICE))
        if recovery:
            cp = cpd[:m * L.n_elim * L.n_keep].cpu().numpy()
            coup[e0:e1] = np.transpose(cp.reshape(m, L.n_keep, L.n_elim), (0, 2, 1))
            erhs[e0:e1] = epd[:m * L.n_elim].cpu().numpy().reshape(m, L.n_elim)
        t_local += t1 - t0
        t_dev += time.perf_counter() - t1
    del mats, rhs
    b = np.zeros(A.n)
    N.check(ctx.lib.pscu_assembly_rhs(ctx.h, A.h, b.ctypes.data, N.PSCU_HOST))
    lay = S.make_layout3(k, mesh.n_faces, mesh.n_elements)
    info = dict(t_local_s=t_local, t_condense_s=t_dev, brow_ptr=brp, bcols=bcols, local=L,
                elim_coupling=coup, elim_rhs=erhs, producer="device")
    return A, b, lay, info


def local_blocks3_device(mesh: Mesh3, k: int, e0: int, e1: int, data: str = "random",
                         seed: int = 0, eta: float = 0.0, ctx=None):
    """The 3D local blocks of elements [e0, e1) built on the device
    (pscu_local_blocks3), host buffers in and out: the same arrays as
    HpLocal3.local_blocks, bit for bit."""
    from . import solver as S

    ctx = ctx or S.default_context()
    L = HpLocal3(k)
    d = mesh.device_inputs(k, data, seed, e0, e1)
    m, n = e1 - e0, L.n_local
    mats, rhs = np.zeros(m * n * n), np.zeros(m * n)
    eta_v = eta if eta > 0.0 else 3.0 * (k + 1) * (k + 1)
    N.check(ctx.lib.pscu_local_blocks3(ctx.h, k, DATA3[data], eta_v, d["nq1"], d["gl"].ctypes.data,
                                       mesh.n_vertices, d["xyz"].ctypes.data, mesh.n_faces,
                                       d["ftab"].ctypes.data, m, d["hex"].ctypes.data,
                                       d["ef"].ctypes.data, d["es"].ctypes.data, N.ptr(d["coef"]),
                                       mats.ctypes.data, rhs.ctypes.data, N.PSCU_HOST))
    return mats, rhs


def assemble_stokes3(mesh: Mesh3, k: int, data: str = "random", seed: int = 0, eta: float = 0.0,
                     batch: int = 4096, nthreads: int = 0, ctx=None, recovery: bool = False,
                     producer: str = "auto"):
    """assemble_hho (assemble.hpp:136-172) for the 3D HHO-hp vp-cond scheme
    into face-block device storage, streamed over element batches: a batch of
    local blocks is built — on the device (pscu_local_blocks3, producer
    "device"; the default for data "zero"/"random") or by the host producer
    ("host", overlapped with the device work; needed for "manufactured") —
    and the device condenses it and scatters the Schur blocks and reduced
    loads (pscu_assembly_add). Both producers give the same blocks bit for
    bit. Returns (A, rhs, layout, info) with A a device CsrMatrix in block
    storage; with recovery the per-element elim_coupling / elim_rhs are
    returned in info."""
    from . import solver as S

    ctx = ctx or S.default_context()
    if producer == "auto":
        producer = "device" if DATA3[data] in (0, 3) else "host"
    if producer == "device":
        return _assemble_stokes3_device(mesh, k, data, seed, eta, batch, ctx, recovery)
    if producer != "host":
        raise ValueError(f"unknown producer {producer!r}")
    L = HpLocal3(k)
    brp, bcols = mesh.block_pattern()
    h = C.c_void_p()
    N.check(ctx.lib.pscu_assembly_begin(ctx.h, mesh.n_faces, L.face_block, brp.ctypes.data,
                                        bcols.ctypes.data, C.byref(h)))
    A = S.CsrMatrix(None, None, None, ctx=ctx, _handle=h.value)
    A._owned = True
    ef = mesh.element_faces()
    keep_pos = np.ascontiguousarray(L.keep_pos, np.int32)
    n = L.n_local
    nb = min(batch, mesh.n_elements)
    # page-locked double buffer: the host builds batch i + 1 while the device
    # condenses and scatters batch i
    pinned = [(N.PinnedArray(nb * n * n), N.PinnedArray(nb * n)) for _ in range(2)]
    bufs = [(pm.a, pr.a) for pm, pr in pinned]
    coup = erhs = None
    if recovery:
        coup = np.empty((mesh.n_elements, L.n_elim, L.n_keep))
        erhs = np.empty((mesh.n_elements, L.n_elim))
    import threading
    import time
    starts = list(range(0, mesh.n_elements, nb))
    t_host = 0.0
    t_dev = 0.0
    err = []

    def build(i):
        nonlocal t_host
        e0 = starts[i]
        e1 = min(mesh.n_elements, e0 + nb)
        t0 = time.perf_counter()
        try:
            L.local_blocks(mesh, e0, e1, data=data, seed=seed, eta=eta, nthreads=nthreads,
                           out=bufs[i % 2])
        except Exception as ex:  # surfaced in the main thread
            err.append(ex)
        t_host += time.perf_counter() - t0

    build(0)
    for i, e0 in enumerate(starts):
        if err:
            raise err[0]
        e1 = min(mesh.n_elements, e0 + nb)
        mats, rhs = bufs[i % 2]
        worker = None
        if i + 1 < len(starts):
            worker = threading.Thread(target=build, args=(i + 1,))
            worker.start()
        t1 = time.perf_counter()
        efb = np.ascontiguousarray(ef[e0:e1], np.int32)
        cp = ep = None
        if recovery:
            cp = np.empty((e1 - e0) * L.n_elim * L.n_keep)
            ep = np.empty((e1 - e0) * L.n_elim)
        N.check(ctx.lib.pscu_assembly_add(ctx.h, A.h, e0, e1 - e0, n, mats.ctypes.data,
                                          rhs.ctypes.data, L.n_elim, L.elim.ctypes.data,
                                          efb.ctypes.data, 6, keep_pos.ctypes.data,
                                          None if cp is None else cp.ctypes.data,
                                          None if ep is None else ep.ctypes.data, N.PSCU_HOST))
        if recovery:
            # column-major ne x nk blocks -> (ne, nk)
            coup[e0:e1] = np.transpose(cp.reshape(e1 - e0, L.n_keep, L.n_elim), (0, 2, 1))
            erhs[e0:e1] = ep.reshape(e1 - e0, L.n_elim)
        t_dev += time.perf_counter() - t1
        if worker is not None:
            worker.join()
    if err:
        raise err[0]
    del bufs, pinned
    b = np.zeros(A.n)
    N.check(ctx.lib.pscu_assembly_rhs(ctx.h, A.h, b.ctypes.data, N.PSCU_HOST))
    lay = S.make_layout3(k, mesh.n_faces, mesh.n_elements)
    info = dict(t_local_s=t_host, t_condense_s=t_dev, brow_ptr=brp, bcols=bcols, local=L,
                elim_coupling=coup, elim_rhs=erhs)
    return A, b, lay, info


def assemble_dg3(mesh: Mesh3, k: int, data: str = "random", seed: int = 0, eta: float = 0.0,
                 batch: int = 2048, nthreads: int = 0, ctx=None):
    """assemble_dg (assemble.hpp:177-346) for the 3D DG scheme (BASELINE.json
    config 4) into DG block device storage: the host producer (C++/OpenMP)
    writes batches of block rows — every entry summed in the reference's
    scatter order — into a page-locked buffer, and each batch is copied into
    the device operator while the next is built. Returns (A, rhs, layout,
    info) with A a device CsrMatrix in DG block storage."""
    import threading
    import time

    from . import solver as S

    ctx = ctx or S.default_context()
    D = DgLocal3(k)
    brp, bcols = D.block_pattern(mesh)
    A = S.dgb_matrix(brp, bcols, None, D.ne, ctx=ctx)
    bsz = 10 * D.ne * D.ne
    ne = mesh.n_elements
    nb = min(batch, ne)
    max_blocks = int(max(brp[min(e0 + nb, ne)] - brp[e0] for e0 in range(0, ne, nb)))
    lib = ctx.lib
    bufs = []
    for _ in range(2):
        p = C.c_void_p()
        N.check(lib.pscu_host_alloc(8 * max_blocks * bsz, C.byref(p)))
        bufs.append(p)
    rhs = np.zeros(ne * D.elem_block)
    t0 = time.perf_counter()
    t_host = 0.0
    try:
        views = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), (max_blocks * bsz,))
                 for p in bufs]
        ranges = [(e0, min(ne, e0 + nb)) for e0 in range(0, ne, nb)]

        def build(i):
            e0, e1 = ranges[i]
            D.rows(mesh, brp, bcols, e0, e1, data=data, seed=seed, eta=eta, nthreads=nthreads,
                   out=(views[i % 2], rhs[e0 * D.elem_block:e1 * D.elem_block]))

        th = None
        err = []

        def run(i):
            try:
                build(i)
            except Exception as ex:  # surfaced after join
                err.append(ex)

        th0 = time.perf_counter()
        build(0)
        t_host += time.perf_counter() - th0
        for i, (e0, e1) in enumerate(ranges):
            if i + 1 < len(ranges):
                N.check(lib.pscu_synchronize(ctx.h))  # buffer (i + 1) % 2 is free again
                th = threading.Thread(target=run, args=(i + 1,))
                th.start()
            q0, q1 = int(brp[e0]), int(brp[e1])
            N.check(lib.pscu_mat_set_values(ctx.h, A.h, q0 * bsz, (q1 - q0) * bsz,
                                            bufs[i % 2].value, N.PSCU_HOST))
            if th is not None:
                th.join()
                th = None
                if err:
                    raise err[0]
    finally:
        for p in bufs:
            lib.pscu_host_free(p)
    lay = S.make_layout3(k, mesh.n_faces, mesh.n_elements, scheme="dg", strategy="uncond")
    info = dict(t_assembly_s=time.perf_counter() - t0, brow_ptr=brp, bcols=bcols, local=D,
                producer="host")
    return A, rhs, lay, info
