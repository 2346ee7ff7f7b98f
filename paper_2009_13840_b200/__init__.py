"""B200-native solver hot path for the pstokes reference (arXiv 2009.13840):
static condensation, condensed-operator SpMV, p-level operator inheritance,
ILU(0)-GMRES smoothed V-cycles and FGMRES, as sm_100a CUDA behind the C ABI
of include/pstokes_cuda.h. See DESIGN.md."""

__all__ = ["solver", "build"]
