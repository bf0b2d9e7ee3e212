"""ctypes binding of libzp.so (the C ABI declared in include/*.h).

The product has no CPU fallback: if the shared library is missing this module
raises at import time, loudly. Build it with ``python -m paper_2408_12596_b200.build``
or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libzp.so")


class ZpLibraryMissing(ImportError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ZpLibraryMissing(
            f"{LIB_PATH} not found: the CUDA extension is not built "
            "(run `python paper_2408_12596_b200/build.py`)")
    return C.CDLL(LIB_PATH)


lib = _load()


class GemmDesc(C.Structure):
    _fields_ = [
        ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("nb1", C.c_int32), ("nb2", C.c_int32),
        ("a", C.c_void_p), ("a_major", C.c_int32), ("lda", C.c_int64), ("a_bs1", C.c_int64), ("a_bs2", C.c_int64),
        ("b", C.c_void_p), ("b_major", C.c_int32), ("ldb", C.c_int64), ("b_bs1", C.c_int64), ("b_bs2", C.c_int64),
        ("c", C.c_void_p), ("ldc", C.c_int64), ("c_bs1", C.c_int64), ("c_bs2", C.c_int64),
        ("alpha", C.c_float),
        ("epilogue", C.c_int32),
        ("causal", C.c_int32),
        ("bias", C.c_void_p),
        ("aux", C.c_void_p),
        ("aux_out", C.c_void_p),
        ("max_ctas", C.c_int32),
        ("split_k", C.c_int32),
        ("colsum", C.c_void_p),
    ]


lib.zp_gemm.argtypes = [C.POINTER(GemmDesc), C.c_void_p]
lib.zp_gemm.restype = C.c_int

lib.zp_launch_count.argtypes = []
lib.zp_launch_count.restype = C.c_int64

lib.zp_attention_fwd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                 C.c_int32, C.c_void_p]
lib.zp_attention_fwd.restype = C.c_int
lib.zp_attention_fwd_hd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_void_p]
lib.zp_attention_fwd_hd.restype = C.c_int
lib.zp_attention_bwd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
lib.zp_attention_bwd.restype = C.c_int
lib.zp_attention_bwd_hd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]
lib.zp_attention_bwd_hd.restype = C.c_int
lib.zp_norm_bwd.argtypes = [C.c_void_p] * 8 + [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                            C.c_int32, C.c_int32, C.c_void_p]
lib.zp_norm_bwd.restype = C.c_int
lib.zp_synth_tokens.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int32, C.c_uint64, C.c_uint64,
                                C.c_void_p]
lib.zp_synth_tokens.restype = C.c_int
