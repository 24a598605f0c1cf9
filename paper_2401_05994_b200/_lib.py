"""ctypes loader for the in-tree sm_100a library ``libmgrc_gpu.so``.

There is deliberately no fallback: if the library is missing or cannot be
loaded, importing the package fails with an explicit error.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmgrc_gpu.so"

P = C.c_void_p
U64P = C.POINTER(C.c_uint64)
IP = C.POINTER(C.c_int)


class ContainerInfoC(C.Structure):
    """mgrc_container_info (include/mgrc_gpu.h)."""

    _fields_ = [
        ("version", C.c_uint16), ("constant_field", C.c_uint8), ("coords_present", C.c_uint8),
        ("dtype", C.c_uint8), ("ndims", C.c_uint8), ("nlevels", C.c_uint8), ("codec_id", C.c_uint8),
        ("shape", C.c_uint64 * 4), ("mode", C.c_uint8), ("norm", C.c_uint8),
        ("smoothness", C.c_double), ("tol", C.c_double), ("bin_widths", C.c_double * 65),
        ("payload_len", C.c_uint64), ("checksum", C.c_uint32), ("header_size", C.c_uint64),
        ("l2_projection", C.c_uint8),
    ]


# every symbol declared in include/mgrc_gpu.h: name -> (restype, argtypes)
SIGNATURES = {
    "mgrc_gpu_compress": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.POINTER(P), U64P]),
    "mgrc_gpu_compress_to": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int,
                                       C.c_int, P, C.c_uint64, U64P]),
    "mgrc_gpu_decompress": (C.c_int, [P, C.c_uint64, C.POINTER(P), IP, IP, P]),
    "mgrc_gpu_compress_l2": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int,
                                       C.POINTER(P), U64P]),
    "mgrc_gpu_compress_l2_to": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int,
                                          C.c_int, P, C.c_uint64, U64P]),
    "mgrc_gpu_host_alloc": (C.c_int, [C.c_uint64, C.POINTER(P)]),
    "mgrc_gpu_host_free": (None, [P]),
    "mgrc_gpu_decompress_into": (C.c_int, [P, C.c_uint64, P, C.c_uint64, IP, IP, P]),
    "mgrc_gpu_inspect": (C.c_int, [P, C.c_uint64, C.POINTER(ContainerInfoC)]),
    "mgrc_gpu_describe": (C.c_int, [P, C.c_uint64, C.POINTER(C.c_char_p)]),
    "mgrc_gpu_plan_chunks": (C.c_int, [C.c_int, P, C.c_int, C.c_uint64, U64P, P, C.c_uint64]),
    "mgrc_gpu_compress_chunked": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int,
                                            C.c_int, C.c_uint64, C.POINTER(P), U64P]),
    "mgrc_gpu_decompress_chunked": (C.c_int, [P, C.c_uint64, C.POINTER(P), IP, IP, P]),
    "mgrc_gpu_compress_chunked_multi": (C.c_int, [P, C.c_int, C.c_int, P, P, C.c_double, C.c_int, C.c_double, C.c_int,
                                                  C.c_int, C.c_uint64, C.c_int, C.POINTER(P), U64P]),
    "mgrc_gpu_decompress_chunked_multi": (C.c_int, [P, C.c_uint64, C.c_int, C.POINTER(P), IP, IP, P]),
    "mgrc_gpu_field_stats": (C.c_int, [P, C.c_int, C.c_uint64, C.POINTER(C.c_double), C.POINTER(C.c_double), IP]),
    "mgrc_gpu_serial_sumsq": (C.c_int, [P, C.c_int, C.c_uint64, C.c_double, C.POINTER(C.c_double)]),
    # MDR (struct arguments as void*; paper_2401_05994_b200/mdr.py binds the structs)
    "mgrc_gpu_mdr_refactor": (C.c_int, [P, C.c_int, P, P, C.c_uint32, C.POINTER(P)]),
    "mgrc_gpu_mdr_store_manifest": (C.c_int, [P, P, P]),
    "mgrc_gpu_mdr_store_segment": (C.c_int, [P, C.c_uint32, C.c_uint32, C.POINTER(P), U64P]),
    "mgrc_gpu_mdr_store_free": (None, [P]),
    "mgrc_gpu_mdr_request": (C.c_int, [P, P, C.c_double, C.c_int, C.c_double, P, P, P, C.c_uint64, U64P, U64P,
                                       C.POINTER(C.c_double), IP]),
    "mgrc_gpu_mdr_session_new": (C.c_int, [P, P, P, C.POINTER(P)]),
    "mgrc_gpu_mdr_reconstruct": (C.c_int, [P, P, P, C.c_uint64, P, P, C.c_int, C.c_double, P,
                                           C.POINTER(C.c_double), P]),
    "mgrc_gpu_mdr_session_free": (None, [P]),
    "mgrc_gpu_last_error": (C.c_char_p, []),
    "mgrc_gpu_free": (None, [P]),
    "mgrc_gpu_set_device": (C.c_int, [C.c_int]),
    "mgrc_gpu_set_stream": (C.c_int, [P]),
    "mgrc_gpu_set_profiling": (C.c_int, [C.c_int]),
    "mgrc_gpu_profile_count": (C.c_int, []),
    "mgrc_gpu_profile_entry": (C.c_int, [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
    "mgrc_gpu_version": (C.c_char_p, []),
    "mgrc_gpu_launch_count": (C.c_uint64, []),
    "mgrc_gpu_nlevels": (C.c_int, [C.c_int, P, P, IP]),
    "mgrc_gpu_initial_bin_widths": (C.c_int, [C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, P]),
    "mgrc_gpu_forward_transform": (C.c_int, [P, C.c_int, P, P, P]),
    "mgrc_gpu_inverse_transform": (C.c_int, [P, C.c_int, P, P, P]),
    "mgrc_gpu_forward_transform_l2": (C.c_int, [P, C.c_int, P, P, P]),
    "mgrc_gpu_inverse_transform_l2": (C.c_int, [P, C.c_int, P, P, P]),
    "mgrc_gpu_quantize": (C.c_int, [P, C.c_int, P, P, P, C.c_int, P, P, U64P]),
    "mgrc_gpu_dequantize": (C.c_int, [P, C.c_int, P, P, P, C.c_int, P]),
    "mgrc_gpu_last_compress_stats": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), IP, IP]),
}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the sm_100a path has no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
