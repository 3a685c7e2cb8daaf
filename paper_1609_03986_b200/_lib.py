"""ctypes binding of include/clatch.h (libclatch.so, built in-tree for sm_100a).

The product has no CPU path: if the shared library is missing, or no B200 is
visible, every compute call raises — nothing falls back to numpy or to oracle/.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libclatch.so"

OK = 0
ERR_INVALID = 1
ERR_CUDA = 2
ERR_NO_DEVICE = 3
ERR_NONFINITE = 5

# 100 + latch::ErrorCode (proj/include/latch/errors.hpp:10-40)
ERROR_NAMES = {
    106: "ImageTooSmall", 107: "TooCloseToBorder", 108: "BadHeader", 109: "BadTripletCount",
    110: "CoordinateOutOfRange", 111: "DegenerateTriplet", 119: "LengthMismatch",
    120: "EmptyGallery",
}


class LatchError(RuntimeError):
    """Mirror of latch::Error (a std::runtime_error; pybind11 surfaces it as RuntimeError,
    proj/tests/python/test_smoke.py:126-136)."""

    def __init__(self, code_name: str, message: str):
        super().__init__(message if message.startswith(code_name) else f"{code_name}: {message}")
        self.code = code_name


class ClatchDeviceError(RuntimeError):
    """The GPU path could not run (no device, CUDA failure, library not built)."""


u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)
i16p = C.POINTER(C.c_int16)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
szp = C.POINTER(C.c_size_t)

_SIGNATURES = {
    "clatch_last_error": (C.c_char_p, []),
    "clatch_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "clatch_ctx_destroy": (None, [C.c_void_p]),
    "clatch_device_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p,
                                     C.c_size_t]),
    "clatch_synchronize": (C.c_int, [C.c_void_p]),
    "clatch_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "clatch_extract_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "clatch_set_pattern": (C.c_int, [C.c_void_p, i16p, C.c_int, C.c_int, f64p]),
    "clatch_descriptor_bytes": (C.c_int, [C.c_void_p]),
    "clatch_prepare_keypoints": (C.c_int, [f64p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_int, f64p,
                                           i64p, szp]),
    "clatch_take_keypoints": (C.c_int, [f64p, C.c_int, i64p, C.c_size_t, C.c_int, f64p]),
    "clatch_detect_u8": (C.c_int, [C.c_void_p, u8p, C.c_int, C.c_int, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                   C.c_int, f64p, C.c_size_t, szp]),
    "clatch_detect_f64": (C.c_int, [C.c_void_p, f64p, C.c_int, C.c_int, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                    C.c_int, f64p, C.c_size_t, szp]),
    "clatch_extract_u8": (C.c_int, [C.c_void_p, u8p, C.c_int, C.c_int, C.c_size_t, f64p, C.c_size_t,
                                    u8p]),
    "clatch_extract_f64": (C.c_int, [C.c_void_p, f64p, C.c_int, C.c_int, C.c_size_t, f64p, C.c_size_t,
                                     u8p]),
    "clatch_describe_all_u8": (C.c_int, [C.c_void_p, u8p, C.c_int, C.c_int, C.c_size_t, f64p, C.c_size_t,
                                         C.c_int, C.c_int, i64p, u8p, szp]),
    "clatch_describe_all_f64": (C.c_int, [C.c_void_p, f64p, C.c_int, C.c_int, C.c_size_t, f64p, C.c_size_t,
                                          C.c_int, C.c_int, i64p, u8p, szp]),
    "clatch_describe_batch_u8": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                           szp, C.POINTER(C.c_void_p), szp, C.c_int, C.c_size_t, C.c_int,
                                           C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), szp]),
    "clatch_describe_batch_f64": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                            szp, C.POINTER(C.c_void_p), szp, C.c_int, C.c_size_t, C.c_int,
                                            C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), szp]),
    "clatch_extract_u8_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_size_t,
                                        C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "clatch_extract_f64_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_size_t,
                                         C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "clatch_estimate_planes_u8_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_size_t,
                                                C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "clatch_match_top2": (C.c_int, [C.c_void_p, u8p, C.c_size_t, u8p, C.c_size_t, C.c_int, i32p, i32p,
                                    i32p]),
    "clatch_match_top2_dev": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                        C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "clatch_filter_matches": (C.c_int, [i32p, i32p, i32p, C.c_size_t, C.c_int, C.c_double, C.c_int,
                                        C.c_int, i32p, i32p, szp]),
    "clatch_match_brute_force": (C.c_int, [C.c_void_p, u8p, C.c_size_t, u8p, C.c_size_t, C.c_int,
                                           C.c_int, C.c_double, C.c_int, C.c_int, C.c_int, i32p, szp]),
    "clatch_triplet_bits": (C.c_int, [C.c_void_p, f64p, C.c_size_t, i16p, C.c_size_t, C.c_int, f64p, u8p,
                                      C.c_size_t]),
    "clatch_set_create": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]),
    "clatch_set_destroy": (None, [C.c_void_p]),
    "clatch_set_count": (C.c_size_t, [C.c_void_p]),
    "clatch_match_sets": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.c_int, i32p, szp]),
    "clatch_match_set_pairs": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_size_t, i32p, C.c_size_t, C.c_int,
                                         C.c_double, C.c_int, C.c_int, C.c_int, i32p, C.c_size_t, szp]),
    "clatch_debug_tc_tile": (C.c_int, [C.c_void_p, u8p, C.c_size_t, u8p, C.c_size_t, i32p, i32p, i32p, i32p]),
    "clatch_launch_count": (C.c_uint64, [C.c_void_p]),
    "clatch_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "clatch_host_free": (C.c_int, [C.c_void_p]),
}

EXPORTS = tuple(_SIGNATURES)

_lib = None


def load():
    """Load libclatch.so (once). Raises ClatchDeviceError if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ClatchDeviceError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or make -C paper_1609_03986_b200/csrc). There is no CPU fallback.")
        lib = C.CDLL(str(LIB_PATH))
        for name, (restype, argtypes) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = restype
            fn.argtypes = argtypes
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = load().clatch_last_error().decode(errors="replace")
    if rc in ERROR_NAMES:
        raise LatchError(ERROR_NAMES[rc], msg)
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_NONFINITE:
        raise LatchError("OutOfBounds", msg)
    raise ClatchDeviceError(msg)
