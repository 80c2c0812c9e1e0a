"""ctypes binding of the C ABI in include/fasth_b200.h.

The product is ``lib/libfasth_b200.so`` (sm_100a kernels + C ABI).  This
module only declares its symbols; there is no fallback: importing the
package without the library, or calling it without a B200, raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# FASTH_LIB selects an alternative in-tree build (tuning variants under lib/variants/)
LIB_PATH = os.environ.get("FASTH_LIB") or os.path.join(HERE, "lib", "libfasth_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fasth_b200.h")

FP = C.POINTER(C.c_float)
I64 = C.c_int64
VP = C.c_void_p


class SvdParamC(C.Structure):
    _fields_ = [("out_dim", C.c_int), ("in_dim", C.c_int), ("nu", C.c_int), ("nv", C.c_int),
                ("U", VP), ("ldu", I64), ("V", VP), ("ldv", I64), ("sigma", VP)]


# name -> (restype, argtypes)
SIGNATURES = {
    "fasth_last_error": (C.c_char_p, []),
    "fasth_version": (C.c_int, []),
    "fasth_ctx_create": (C.c_int, [C.c_int, VP, C.POINTER(VP)]),
    "fasth_ctx_destroy": (C.c_int, [VP]),
    "fasth_ctx_set_stream": (C.c_int, [VP, VP]),
    "fasth_ctx_set_check": (C.c_int, [VP, C.c_int]),
    "fasth_ctx_check": (C.c_int, [VP]),
    "fasth_ctx_launch_count": (I64, [VP]),
    "fasth_ctx_trim": (C.c_int, [VP]),
    "fasth_ctx_set_dv_events": (C.c_int, [VP, C.POINTER(VP), C.c_int]),
    "fasth_ctx_dv_buckets": (C.c_int, [VP, C.POINTER(I64), C.c_int]),
    "fasth_device_alloc": (C.c_int, [VP, I64, C.POINTER(VP)]),
    "fasth_device_free": (C.c_int, [VP, VP]),
    "fasth_copy": (C.c_int, [VP, VP, VP, I64, C.c_int]),
    "fasth_ctx_synchronize": (C.c_int, [VP]),
    "fasth_ctx_set_timing": (C.c_int, [VP, C.c_int]),
    "fasth_ctx_kernel_times": (C.c_int, [VP, C.c_char_p, C.c_int]),
    "fasth_forward": (C.c_int, [VP, VP, I64, C.c_int, C.c_int, VP, I64, C.c_int, C.c_int, VP, I64,
                                C.POINTER(VP)]),
    "fasth_backward": (C.c_int, [VP, VP, VP, I64, VP, I64, VP, I64]),
    "fasth_tape_destroy": (C.c_int, [VP]),
    "fasth_tape_info": (C.c_int, [VP] + [C.POINTER(C.c_int)] * 5),
    "fasth_forward_backward": (C.c_int, [VP, VP, I64, C.c_int, C.c_int, VP, I64, VP, I64, C.c_int,
                                         C.c_int, VP, I64, VP, I64, VP, I64]),
    "fasth_forward_backward_host": (C.c_int, [VP, VP, C.c_int, C.c_int, VP, VP, C.c_int, C.c_int,
                                              VP, VP, VP]),
    "fasth_svd_forward": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, C.c_int, C.c_int, VP, I64,
                                    C.POINTER(VP)]),
    "fasth_svd_backward": (C.c_int, [VP, C.POINTER(SvdParamC), VP, VP, I64, VP, I64, VP, I64, VP,
                                     I64, VP]),
    "fasth_svd_forward_backward": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, VP, I64, C.c_int, C.c_int, VP,
                                             I64, VP, I64, VP, I64, VP, I64, VP]),
    "fasth_svd_plan_create": (C.c_int, [VP, C.POINTER(SvdParamC), C.c_int, C.c_int, C.c_int, C.POINTER(VP)]),
    "fasth_svd_plan_destroy": (C.c_int, [VP]),
    "fasth_svd_forward_planned": (C.c_int, [VP, C.POINTER(SvdParamC), VP, VP, I64, C.c_int, C.c_int, VP, I64,
                                            C.POINTER(VP)]),
    "fasth_svd_tape_destroy": (C.c_int, [VP]),
    "fasth_svd_step": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, VP, I64, VP, C.c_float,
                                 C.c_float, VP, I64, VP, I64, VP]),
    "fasth_clamp_sigma": (C.c_int, [VP, VP, C.c_int, C.c_float, VP]),
    "fasth_apply_inverse": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, C.c_int, C.c_int, VP, I64]),
    "fasth_apply_exponential": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, C.c_int, C.c_int, VP,
                                          I64]),
    "fasth_apply_cayley": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, C.c_int, C.c_int, VP, I64]),
    "fasth_svd_file_info": (C.c_int, [C.c_char_p] + [C.POINTER(C.c_int)] * 4),
    "fasth_svd_load": (C.c_int, [VP, C.c_char_p, VP, I64, VP, I64, VP]),
    "fasth_svd_save": (C.c_int, [VP, C.POINTER(SvdParamC), C.c_char_p]),
    "fasth_tune_block_width": (C.c_int, [VP, C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_int)]),
    "fasth_log_abs_det": (C.c_int, [VP, C.POINTER(SvdParamC), C.POINTER(C.c_double)]),
    "fasth_apply_pseudo_inverse": (C.c_int, [VP, C.POINTER(SvdParamC), VP, I64, C.c_int, C.c_double, C.c_int, VP,
                                             I64]),
    "fasth_wy_compact": (C.c_int, [VP, VP, I64, C.c_int, C.c_int, VP, I64, VP, I64]),
    "fasth_compact_chain": (C.c_int, [VP, VP, I64, C.c_int, C.c_int, C.c_int, VP, I64, VP, I64]),
    "fasth_wy_apply": (C.c_int, [VP, VP, I64, VP, I64, C.c_int, C.c_int, VP, I64, C.c_int, VP, I64]),
    "fasth_wy_apply_transpose": (C.c_int, [VP, VP, I64, VP, I64, C.c_int, C.c_int, VP, I64, C.c_int, VP, I64]),
}


def header_symbols(path: str = HEADER) -> list[str]:
    """Every function the public header declares (for the export test)."""
    txt = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:fasth_status|const char\*|int|int64_t)\s+(fasth_\w+)\s*\(",
                                 txt, re.M)))


_lib = None


def load(path: str = LIB_PATH):
    """Load and declare the library (cached).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `make lib` (or __graft_entry__.build())."
                           " There is no CPU fallback.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
