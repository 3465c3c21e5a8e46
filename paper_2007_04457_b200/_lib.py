"""ctypes binding of the C ABI in include/hgr_cuda.h (libhgr_b200.so).

There is deliberately no fallback: if the CUDA library is missing the import
fails loudly. Build it with ``__graft_entry__.build()`` or
``make -C paper_2007_04457_b200/csrc``.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# HGR_B200_LIB: load another build of the same library (A/B timing of variants)
LIB_PATH = Path(os.environ.get("HGR_B200_LIB") or
                Path(__file__).resolve().parent / "lib" / "libhgr_b200.so")

HGR_OK, HGR_ERR_INVALID, HGR_ERR_CUDA, HGR_ERR_NONFINITE, HGR_ERR_NOMEM = 0, 1, 2, 3, 4
HGR_F32, HGR_F64 = 0, 1


class GridDesc(C.Structure):
    _fields_ = [("rank", C.c_int), ("extents", C.c_size_t * 3), ("coords", C.c_void_p * 3)]


class HgInfo(C.Structure):
    """hgr_hg_info = HgFileHeader (storage.hpp:36-55)."""
    _fields_ = [("version", C.c_uint), ("precision_bytes", C.c_uint), ("rank", C.c_int),
                ("extents", C.c_size_t * 3), ("class_count", C.c_int),
                ("header_bytes", C.c_uint64), ("file_bytes", C.c_uint64)]


_vp, _sz, _int = C.c_void_p, C.c_size_t, C.c_int
_G = C.POINTER(GridDesc)

_SIGS = {
    "hgr_cuda_last_error": (C.c_char_p, []),
    "hgr_cuda_abi_version": (_int, []),
    "hgr_cuda_plan_create": (_int, [_G, _int, C.POINTER(_vp)]),
    "hgr_cuda_plan_destroy": (None, [_vp]),
    "hgr_cuda_plan_levels": (_int, [_vp]),
    "hgr_cuda_plan_workspace_bytes": (_sz, [_vp]),
    "hgr_cuda_plan_launches": (_int, [_vp, _int, _int]),
    "hgr_cuda_plan_decompose": (_int, [_vp, _vp, _vp]),
    "hgr_cuda_plan_decompose_to": (_int, [_vp, _vp, _vp, _vp]),
    "hgr_cuda_plan_recompose": (_int, [_vp, _vp, _vp, _int, _vp]),
    "hgr_cuda_plan_sync_status": (_int, [_vp, _vp]),
    "hgr_cuda_plan_set_profiling": (_int, [_vp, _int]),
    "hgr_cuda_plan_read_profile": (_int, [_vp, _vp, _vp, _vp]),
    "hgr_cuda_plan_autotune": (_int, [_vp, _vp, _vp, _vp, C.c_char_p, _sz, C.POINTER(_sz)]),
    "hgr_cuda_plan_reset_tuning": (_int, [_vp]),
    "hgr_cuda_synthetic_field_f64": (_int, [_G, _vp, C.c_ulonglong, _vp, _vp, _vp, _vp]),
    "hgr_cuda_synthetic_field_f32": (_int, [_G, _vp, C.c_ulonglong, _vp, _vp, _vp, _vp]),
    "hgr_class_node_count": (_sz, [_G, _int]),
    "hgr_levels": (_int, [_G]),
    "hgr_hg_read_info": (_int, [C.c_char_p, C.POINTER(HgInfo)]),
    "hgr_hg_read_coords": (_int, [C.c_char_p, _int, _vp]),
    "hgr_hg_read_class_table": (_int, [C.c_char_p, _vp, _vp, _int]),
}
for _t in ("f64", "f32"):
    _SIGS.update({
        f"hgr_cuda_decompose_{_t}": (_int, [_G, _vp, _vp]),
        f"hgr_cuda_decompose_to_{_t}": (_int, [_G, _vp, _vp, _vp]),
        f"hgr_cuda_recompose_{_t}": (_int, [_G, _vp, _vp, _int, _vp]),
        f"hgr_decompose_host_{_t}": (_int, [_G, _vp]),
        f"hgr_recompose_host_{_t}": (_int, [_G, _vp, _vp, _int]),
        f"hgr_cuda_interpolate_to_fine_{_t}": (_int, [_G, _int, _vp, _vp, _vp]),
        f"hgr_cuda_compute_coefficients_{_t}": (_int, [_G, _int, _vp, _vp, _vp]),
        f"hgr_cuda_compute_correction_{_t}": (_int, [_G, _int, _vp, _vp, _vp]),
        f"hgr_cuda_extract_class_{_t}": (_int, [_G, _vp, _int, _vp, _vp]),
        f"hgr_cuda_scatter_class_{_t}": (_int, [_G, _vp, _int, _vp, _vp]),
        f"hgr_cuda_masstrans_apply_{_t}": (_int, [_sz, _sz, _vp, _vp, _vp, _vp]),
        f"hgr_cuda_mass_apply_{_t}": (_int, [_sz, _sz, _vp, _vp, _vp, _vp]),
        f"hgr_cuda_transfer_apply_{_t}": (_int, [_sz, _sz, _vp, _vp, _vp, _vp]),
        f"hgr_cuda_error_report_{_t}": (_int, [_sz, _vp, _vp, _vp, _vp]),
        f"hgr_masstrans_taps_{_t}": (_int, [_sz, _vp, _vp]),
        f"hgr_thomas_factors_{_t}": (_int, [_sz, _vp, _vp, _vp, _vp]),
        f"hgr_host_level_op_{_t}": (_int, [_G, _int, _int, _vp, _vp]),
        f"hgr_host_fiber_op_{_t}": (_int, [_int, _sz, _sz, _vp, _vp, _vp]),
        f"hgr_cuda_apply_coefficients_{_t}": (_int, [_G, _int, _vp, _vp, _vp, _vp]),
        f"hgr_host_apply_coefficients_{_t}": (_int, [_G, _int, _vp, _vp, _vp]),
        f"hgr_error_report_host_{_t}": (_int, [_sz, _vp, _vp, _vp]),
        f"hgr_write_hg_host_{_t}": (_int, [C.c_char_p, _G, _vp, C.POINTER(C.c_uint64)]),
        f"hgr_read_hg_prefix_host_{_t}": (_int, [C.c_char_p, _int, _vp, C.POINTER(C.c_uint64)]),
        f"hgr_cuda_thomas_solve_{_t}": (_int, [_sz, _sz, _vp, _vp, _vp, _vp]),
        f"hgr_cuda_write_hg_{_t}": (_int, [C.c_char_p, _G, _vp, C.POINTER(C.c_uint64), _vp]),
        f"hgr_cuda_read_hg_prefix_{_t}": (_int, [C.c_char_p, _int, _vp, C.POINTER(C.c_uint64),
                                                   _vp]),
    })

EXPORTED_SYMBOLS = tuple(sorted(_SIGS))

_lib = None


def load() -> C.CDLL:
    """Load libhgr_b200.so (raises if it was not built -- no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"hgr CUDA library not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().hgr_cuda_last_error().decode()
