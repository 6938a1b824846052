"""ctypes binding of the C ABI in include/dmm_gpu.h (libdmm_b200.so, built in-tree).

There is no fallback: if the library is missing, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# DMM_B200_LIB: an alternative build of the same library (A/B timing of build variants)
LIB_PATH = os.environ.get("DMM_B200_LIB") or os.path.join(PKG, "libdmm_b200.so")


class GeneralStats(C.Structure):  # dmm_general_stats
    _fields_ = [("cleanup_retries", C.c_uint32), ("sorted", C.c_uint32)]


class PermuteReport(C.Structure):  # dmm_permute_report
    _fields_ = [("iterations", C.c_uint32), ("fallback", C.c_uint32), ("used_packing", C.c_uint32),
                ("packed_width", C.c_uint32), ("threshold", C.c_uint64), ("random_words", C.c_uint64),
                ("cleanup_retries", C.c_uint32), ("n_hist", C.c_uint32)]


# Every symbol include/dmm_gpu.h declares, with its ctypes signature.
_vp, _u32, _u64, _int = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
SIGNATURES = {
    "dmm_version": (C.c_char_p, []),
    "dmm_last_error": (C.c_char_p, []),
    "dmm_supported": (_int, [C.c_char_p, _u32, _u32]),
    "dmm_last_launch_count": (_u32, []),
    "dmm_gen_instances": (_int, [_int, _u32, _u32, _u64, _u64, _vp, _vp]),
    "dmm_gen_keys": (_int, [_u64, _u64, _vp, _vp]),
    "dmm_partition_general": (_int, [_vp, _vp, _u32, _u32, _u64, _u32, _vp, _vp, _vp]),
    "dmm_integer_sort_general": (_int, [_vp, _vp, _u32, _u32, _u64, _u64, _u32, _vp, _vp, _vp]),
    "dmm_general_probe_snaps": (_u32, [_u32, _u32, _u32]),
    "dmm_partition_general_probe": (_int, [_vp, _vp, _u32, _u32, _u64, _u32, _vp, _vp, _vp, _u32, _vp]),
    "dmm_integer_sort_general_probe": (_int, [_vp, _vp, _u32, _u32, _u64, _u64, _u32, _vp, _vp, _vp, _u32, _vp]),
    "dmm_short_wide_probe": (_int, [_vp, _vp, _u32, _u32, _u64, _int, _int, _vp, _vp, _vp]),
    "dmm_permute_steps": (_int, [_vp, _u32, _u32, _u64, _vp, _u32, _u32, _vp, _vp]),
    "dmm_partition_square": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _vp]),
    "dmm_partition_short_wide": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _vp]),
    "dmm_sort_short_wide": (_int, [_vp, _vp, _u32, _u32, _u64, _int, _vp]),
    "dmm_sort_square": (_int, [_vp, _vp, _u32, _u32, _u64, _int, _vp]),
    "dmm_sort_tall": (_int, [_vp, _vp, _u32, _u32, _u64, _vp]),
    "dmm_sort_wide_any": (_int, [_vp, _vp, _u32, _u32, _u64, _int, _vp]),
    "dmm_transpose_square": (_int, [_vp, _vp, _u32, _u64, _vp]),
    "dmm_to_column_major": (_int, [_vp, _vp, _u32, _u32, _u64, _vp]),
    "dmm_to_row_major": (_int, [_vp, _vp, _u32, _u32, _u64, _vp]),
    "dmm_sort_rows": (_int, [_vp, _vp, _u32, _u32, _u64, _int, _u64, _vp, _vp]),
    "dmm_permute_workspace_bytes": (_u64, [_u32, _u32, _u64]),
    "dmm_permute": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _u32, _u32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "dmm_multisplit_workspace_bytes": (_u64, [_u64, _u32]),
    "dmm_multisplit": (_int, [_vp, _u64, _u32, _u32, _vp, _vp, _vp, _vp]),
    "dmm_permute_from_state": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _u32, _u32, _vp, _vp, _vp, _vp, _vp]),
    "dmm_modelled_steps": (_u64, [C.c_char_p, _u32, _u32]),
    "dmm_leaf_steps": (_int, [_vp, _u32, _u32, _u64, _u64, _vp, _vp]),
    "dmm_sort_steps": (_int, [C.c_char_p, _vp, _u32, _u32, _u64, _vp, _vp]),
    "dmm_general_steps": (_int, [_vp, _u32, _u32, _u64, _u64, _vp, _vp, _vp]),
    "dmm_multisplit_count": (_int, [_vp, _u64, _u32, _u32, _vp, _vp, _vp]),
    "dmm_multisplit_scatter_to": (_int, [_vp, _u64, _u32, _u32, _vp, _vp, _vp, _vp]),
    "dmm_offline_schedule": (_int, [_u32, _u32, _vp, _vp]),
    "dmm_apply_schedule_smem_bytes": (_u64, [_u32, _u32, _u32]),
    "dmm_apply_schedule": (_int, [_vp, _vp, _u32, _u32, _u64, _vp, _vp, _u32, _u32, _vp, _vp]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA extension first "
            "(python -m paper_1507_01391_b200.build or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
