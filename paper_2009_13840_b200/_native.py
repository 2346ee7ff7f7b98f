"""ctypes binding of libpstokes_b200.so (include/pstokes_cuda.h).

There is no CPU fallback: importing the solver API on a machine without the
built library or without an sm_100 GPU raises, by design.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import LIB

PSCU_HOST, PSCU_DEVICE = 0, 1

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

EXPORTS = [
    "pscu_last_error", "pscu_version", "pscu_create", "pscu_destroy", "pscu_synchronize",
    "pscu_launch_count", "pscu_timer_start", "pscu_timer_stop", "pscu_profile",
    "pscu_profile_read", "pscu_mat_create", "pscu_mat_destroy", "pscu_mat_dims",
    "pscu_mat_download", "pscu_spmv", "pscu_ilu0_create", "pscu_ilu0_destroy",
    "pscu_ilu0_factors", "pscu_ilu0_apply", "pscu_layout_make", "pscu_layout_dim",
    "pscu_coarse_to_fine", "pscu_inherit", "pscu_gmres", "pscu_fgmres", "pscu_hier_create",
    "pscu_hier_destroy", "pscu_hier_nlev", "pscu_hier_level_mat", "pscu_hier_level_ilu",
    "pscu_vcycle", "pscu_hier_coarse_its", "pscu_hier_reset", "pscu_solve", "pscu_solve_system",
    "pscu_condense_batch", "pscu_condense_assemble", "pscu_recover_batch", "pscu_bj_create",
    "pscu_bj_destroy", "pscu_bj_apply", "pscu_layout_make3", "pscu_bsr_create",
    "pscu_mat_block_size", "pscu_assembly_begin", "pscu_assembly_add", "pscu_assembly_rhs",
    "pscu_solve_system_bsr", "pscu_bsr_download", "pscu_dgb_create", "pscu_mat_dg_modes",
    "pscu_mat_set_values", "pscu_solve_system_dgb", "pscu_host_alloc", "pscu_host_free",
    "pscu_bsr_create_local", "pscu_assembly_begin_local", "pscu_assembly_add_local",
    "pscu_error_accumulate", "pscu_local_blocks3", "pscu_create_devices",
]


class Layout(C.Structure):
    _fields_ = [(f, C.c_int) for f in ("scheme", "strategy", "k", "n_faces", "n_elements",
                                       "face_vel", "face_press", "elem_vel", "elem_press",
                                       "dim")]


class LevelCfg(C.Structure):
    _fields_ = [("smoother", C.c_int), ("smoother_iters", C.c_int), ("coarse", C.c_int),
                ("coarse_rtol", C.c_double), ("coarse_maxit", C.c_int)]


class Report(C.Structure):
    _fields_ = [("outer_its", C.c_int), ("coarse_its", C.c_longlong), ("vcycles", C.c_int),
                ("rel_residual", C.c_double), ("converged", C.c_int), ("t_setup", C.c_double),
                ("t_solve", C.c_double)]


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


_lib = None


def load(path: str = LIB):
    """Loads the native library (raises if it is missing). PSCU_LIB overrides
    the path (experimental builds in tools/)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("PSCU_LIB", path)
    if not os.path.exists(path):
        raise RuntimeError(f"native solver library missing: {path} (run __graft_entry__.build())")
    lib = C.CDLL(path)
    vp, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int, C.c_double
    pi, pd = C.POINTER(C.c_int), C.POINTER(C.c_double)
    lib.pscu_last_error.restype = C.c_char_p
    lib.pscu_create.argtypes = [i32, C.POINTER(vp)]
    lib.pscu_create_devices.argtypes = [C.POINTER(i32), i32, C.POINTER(vp)]
    lib.pscu_destroy.argtypes = [vp]
    lib.pscu_synchronize.argtypes = [vp]
    lib.pscu_launch_count.restype = C.c_longlong
    lib.pscu_launch_count.argtypes = [vp]
    lib.pscu_timer_start.argtypes = [vp]
    lib.pscu_timer_stop.argtypes = [vp, pd]
    lib.pscu_profile.argtypes = [vp, i32]
    lib.pscu_profile_read.argtypes = [vp, i32, C.POINTER(C.c_longlong), pd, pd]
    lib.pscu_mat_create.argtypes = [vp, i64, vp, vp, vp, i32, C.POINTER(vp)]
    lib.pscu_mat_destroy.argtypes = [vp]
    lib.pscu_mat_dims.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
    lib.pscu_mat_download.argtypes = [vp, vp, vp, vp, vp]
    lib.pscu_spmv.argtypes = [vp, vp, vp, vp, i32]
    lib.pscu_ilu0_create.argtypes = [vp, vp, C.POINTER(vp)]
    lib.pscu_ilu0_destroy.argtypes = [vp]
    lib.pscu_ilu0_factors.argtypes = [vp, vp, vp]
    lib.pscu_ilu0_apply.argtypes = [vp, vp, vp, vp, i32]
    lib.pscu_bj_create.argtypes = [vp, vp, C.POINTER(Layout), C.POINTER(vp)]
    lib.pscu_bj_destroy.argtypes = [vp]
    lib.pscu_bj_apply.argtypes = [vp, vp, vp, vp, i32]
    lib.pscu_layout_make.argtypes = [i32, i32, i32, i32, i32, C.POINTER(Layout)]
    lib.pscu_layout_dim.restype = i64
    lib.pscu_layout_dim.argtypes = [C.POINTER(Layout)]
    lib.pscu_coarse_to_fine.argtypes = [C.POINTER(Layout), C.POINTER(Layout), vp]
    lib.pscu_inherit.argtypes = [vp, vp, C.POINTER(Layout), C.POINTER(Layout), C.POINTER(vp)]
    lib.pscu_gmres.argtypes = [vp, vp, vp, vp, vp, i32, f64, i32, vp, pi, pd, pi, i32]
    lib.pscu_fgmres.argtypes = [vp, vp, vp, vp, i32, f64, vp, pi, pd, pi, i32]
    lib.pscu_hier_create.argtypes = [vp, vp, C.POINTER(Layout), vp, i32, C.POINTER(LevelCfg),
                                     C.POINTER(vp)]
    lib.pscu_hier_destroy.argtypes = [vp]
    lib.pscu_hier_nlev.argtypes = [vp]
    lib.pscu_hier_level_mat.restype = vp
    lib.pscu_hier_level_mat.argtypes = [vp, i32]
    lib.pscu_hier_level_ilu.restype = vp
    lib.pscu_hier_level_ilu.argtypes = [vp, i32]
    lib.pscu_vcycle.argtypes = [vp, vp, i32, vp, vp, i32]
    lib.pscu_hier_coarse_its.restype = C.c_longlong
    lib.pscu_hier_coarse_its.argtypes = [vp]
    lib.pscu_hier_reset.argtypes = [vp]
    lib.pscu_solve.argtypes = [vp, vp, vp, f64, i32, i32, vp, vp, C.POINTER(Report), i32]
    lib.pscu_solve_system.argtypes = [vp, i64, vp, vp, vp, vp, C.POINTER(Layout), vp, i32,
                                      C.POINTER(LevelCfg), f64, i32, i32, vp, vp,
                                      C.POINTER(Report)]
    lib.pscu_condense_batch.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, vp, vp, vp, pi, i32]
    lib.pscu_condense_assemble.argtypes = [vp, i32, i32, vp, vp, i32, vp, vp, i64, vp, vp,
                                           C.POINTER(Layout), i32, C.POINTER(vp), vp, vp, vp]
    lib.pscu_recover_batch.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32]
    lib.pscu_error_accumulate.argtypes = [vp, vp, i32, vp, vp, vp, i32]
    lib.pscu_local_blocks3.argtypes = [vp, i32, i32, f64, i32, vp, i64, vp, i64, vp, i32, vp, vp, vp,
                                       vp, vp, vp, i32]
    lib.pscu_layout_make3.argtypes = [i32, i32, i32, i32, i32, C.POINTER(Layout)]
    lib.pscu_bsr_create.argtypes = [vp, i64, i32, vp, vp, vp, i32, C.POINTER(vp)]
    lib.pscu_mat_block_size.argtypes = [vp]
    lib.pscu_dgb_create.argtypes = [vp, i64, i32, vp, vp, vp, i32, C.POINTER(vp)]
    lib.pscu_mat_dg_modes.argtypes = [vp]
    lib.pscu_mat_set_values.argtypes = [vp, vp, i64, i64, vp, i32]
    lib.pscu_bsr_download.argtypes = [vp, vp, vp, vp, vp]
    lib.pscu_host_alloc.argtypes = [i64, C.POINTER(vp)]
    lib.pscu_bsr_create_local.argtypes = [vp, i64, i64, i32, i64, vp, vp, vp, i32, C.POINTER(vp)]
    lib.pscu_assembly_begin_local.argtypes = [vp, i64, i64, i32, i64, vp, vp, C.POINTER(vp)]
    lib.pscu_assembly_add_local.argtypes = [vp, vp, i32, i32, i32, vp, vp, i32, vp, vp, vp, i32,
                                            vp, i32]
    lib.pscu_host_free.argtypes = [vp]
    lib.pscu_assembly_begin.argtypes = [vp, i64, i32, vp, vp, C.POINTER(vp)]
    lib.pscu_assembly_add.argtypes = [vp, vp, i32, i32, i32, vp, vp, i32, vp, vp, i32, vp, vp,
                                      vp, i32]
    lib.pscu_assembly_rhs.argtypes = [vp, vp, vp, i32]
    lib.pscu_solve_system_bsr.argtypes = [vp, i64, i32, vp, vp, vp, vp, C.POINTER(Layout), vp,
                                          i32, C.POINTER(LevelCfg), f64, i32, i32, vp, vp,
                                          C.POINTER(Report)]
    lib.pscu_solve_system_dgb.argtypes = lib.pscu_solve_system_bsr.argtypes
    _lib = lib
    return lib


def check(rc: int):
    if rc != 0:
        msg = load().pscu_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise NativeError(rc, msg)


def ptr(a) -> int | None:
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class PinnedArray:
    """A page-locked host float64 array (pscu_host_alloc) viewed as numpy."""

    def __init__(self, count: int):
        self.lib = load()
        p = C.c_void_p()
        check(self.lib.pscu_host_alloc(8 * max(count, 1), C.byref(p)))
        self.p = p
        buf = (C.c_double * max(count, 1)).from_address(p.value)
        self.a = np.frombuffer(buf, dtype=np.float64, count=count)

    def __del__(self):
        if getattr(self, "p", None):
            self.a = None
            self.lib.pscu_host_free(self.p)
            self.p = None
