"""ctypes binding of the in-tree C-ABI library ``libfgc_b200.so``.

This is the only way the Python package reaches the GPU; there is no CPU or
numpy fallback.  If the library is missing the import fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# FGC_LIB_VARIANT=x loads libfgc_b200.x.so (A/B builds of the same tree)
LIB_PATH = _HERE / ("libfgc_b200.%s.so" % os.environ["FGC_LIB_VARIANT"]
                    if os.environ.get("FGC_LIB_VARIANT") else "libfgc_b200.so")

OK = 0
ERR_INVALID, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL = 1, 2, 3, 4
ERR_HEADER, ERR_TRUNCATED, ERR_BITMAP, ERR_FORMAT, ERR_NO_CONFIG = 5, 6, 7, 8, 9

FLAG_NONFINITE, FLAG_HALF_OVERFLOW, FLAG_F32_RANGE, FLAG_CAPACITY = 1, 2, 4, 8
MODE_COUNT, MODE_ENERGY = 0, 1
DTYPE_F32, DTYPE_F64 = 0, 1
HEADER_BYTES = 36
MAX_WORKERS = 256


class Quantizer(C.Structure):
    _fields_ = [("min", C.c_float), ("max", C.c_float), ("eps", C.c_float),
                ("n_bits", C.c_int32), ("mantissa_bits", C.c_int32), ("pbase", C.c_uint32),
                ("pos_count", C.c_uint32), ("neg_count", C.c_uint32),
                ("actual_min", C.c_float), ("actual_max", C.c_float)]


class CodecDesc(C.Structure):
    _fields_ = [("n", C.c_uint64), ("chunk_size", C.c_uint32), ("mode", C.c_int32),
                ("theta", C.c_double), ("half_pass", C.c_int32), ("passthrough", C.c_int32),
                ("full_capacity", C.c_int32), ("quant", Quantizer)]


class PlanInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("n_chunks", C.c_uint32), ("chunk_size", C.c_uint32),
                ("tail_len", C.c_uint32), ("n_bits", C.c_uint32), ("message_bytes", C.c_uint64),
                ("wire_bytes_max", C.c_uint64), ("spectrum_bins", C.c_uint64),
                ("fused_chunks", C.c_uint32), ("max_slots", C.c_uint32), ("total_slots", C.c_uint64)]


P = C.c_void_p
U8P = C.POINTER(C.c_uint8)
U32, U64, I32, F64 = C.c_uint32, C.c_uint64, C.c_int, C.c_double

# name -> (restype, argtypes)
_SIGS = {
    "fgc_quantizer_from_params": (I32, [F64, F64, I32, I32, F64, C.POINTER(Quantizer)]),
    "fgc_quantizer_validate": (I32, [C.POINTER(Quantizer)]),
    "fgc_tune_eps": (I32, [F64, F64, I32, I32, F64, C.POINTER(Quantizer)]),
    "fgc_message_layout": (I32, [C.POINTER(CodecDesc), C.POINTER(U32), C.POINTER(U64), P]),
    "fgc_plan_create": (I32, [C.POINTER(CodecDesc), C.POINTER(P)]),
    "fgc_plan_destroy": (None, [P]),
    "fgc_plan_get_info": (I32, [P, C.POINTER(PlanInfo)]),
    "fgc_plan_segment_offsets": (I32, [P, P]),
    "fgc_plan_bin_offsets": (I32, [P, P]),
    "fgc_plan_set_theta": (I32, [P, F64, P]),
    "fgc_compress": (I32, [P, P, I32, P, P, P]),
    "fgc_encode_spectrum": (I32, [P, P, P, P, P, P]),
    "fgc_forward_spectrum": (I32, [P, P, I32, P, P, P]),
    "fgc_decode_average": (I32, [P, P, I32, U64, P, P, P]),
    "fgc_decode_spectrum": (I32, [P, P, I32, U64, P, P, P]),
    "fgc_inverse_spectrum": (I32, [P, P, P, P]),
    "fgc_spectrum_error": (I32, [P, P, P, P, P]),
    "fgc_serialize": (I32, [P, P, P, P, P]),
    "fgc_parse_header": (I32, [P, U64, C.POINTER(CodecDesc)]),
    "fgc_wire_index": (I32, [P, U64, C.POINTER(CodecDesc), P, P, C.POINTER(U32)]),
    "fgc_deserialize": (I32, [P, P, P, P, P, P]),
    "fgc_message_counts": (I32, [P, P, P, P]),
    "fgc_message_unpack": (I32, [P, P, P, P, P, P]),
    "fgc_message_pack": (I32, [P, P, P, P, P, P, P, P]),
    "fgc_quantize": (I32, [C.POINTER(Quantizer), P, I32, U64, P, P, P]),
    "fgc_dequantize": (I32, [C.POINTER(Quantizer), P, U64, P, P, P]),
    "fgc_pack_bits": (I32, [P, U64, I32, P, P]),
    "fgc_unpack_bits": (I32, [P, U64, I32, P, P]),
    "fgc_flags_to_bitmap": (I32, [P, U64, P, P]),
    "fgc_bitmap_to_flags": (I32, [P, U64, P, P]),
    "fgc_prefix_sum": (I32, [P, U64, P, P, P, P]),
    "fgc_compact": (I32, [P, P, P, U64, I32, P, P]),
    "fgc_expand": (I32, [P, P, P, U64, I32, P, P]),
    "fgc_rfft": (I32, [P, I32, U64, P, P, P]),
    "fgc_irfft": (I32, [P, U64, P, P]),
    "fgc_truncate": (I32, [P, U64, F64, P, P, P]),
    "fgc_truncate_mode": (I32, [P, U64, U64, F64, I32, P, P, P]),
    "fgc_spectrum_peak": (I32, [P, I32, U64, P, P, P]),
    "fgc_half_round_trip": (I32, [P, U64, P, P]),
    "fgc_nccl_unique_id": (I32, [P]),
    "fgc_nccl_comm_create": (I32, [P, I32, I32, C.POINTER(P)]),
    "fgc_nccl_comm_destroy": (I32, [P]),
    "fgc_allgather": (I32, [P, P, P, U64, P]),
    "fgc_allreduce_sum_f32": (I32, [P, P, U64, P]),
    "fgc_allgather_average": (I32, [P, P, I32, P, I32, P, P, P, P, P, P]),
    "fgc_exchange_create": (I32, [I32, I32, U64, C.POINTER(P)]),
    "fgc_exchange_handles": (I32, [P, P]),
    "fgc_exchange_open": (I32, [P, P]),
    "fgc_exchange_destroy": (None, [P]),
    "fgc_exchange_message": (I32, [P, I32, C.POINTER(P), C.POINTER(P)]),
    "fgc_exchange_average": (I32, [P, P, P, I32, P, P, P, P]),
    "fgc_average_host": (I32, [P, P, P, I32, P, P, P, P, P, P, P]),
    "fgc_profile_fused_compress": (I32, [P, P, I32, P, P, P, P]),
    "fgc_last_error": (C.c_char_p, []),
    "fgc_version": (I32, []),
    "fgc_kernel_launches": (U64, []),
}

EXPORTED = tuple(_SIGS)


def _load():
    if not LIB_PATH.exists():
        if os.environ.get("FGC_AUTOBUILD", "1") == "1":
            from .build import build
            build()
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1811_08596_b200.build`")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


class _Lazy:
    """Loads the library on first use so `python -m paper_1811_08596_b200.build`
    works before the .so exists."""

    _lib = None

    def __getattr__(self, name):
        if _Lazy._lib is None:
            _Lazy._lib = _load()
        return getattr(_Lazy._lib, name)


lib = _Lazy()


class CodecFormatError(ValueError):
    """Malformed compressed data (codec.py:76-77)."""


class CorruptHeaderError(CodecFormatError):
    """Header failed validation (codec.py:80-81)."""


class TruncatedPayloadError(CodecFormatError):
    """Buffer ended before the declared payload was complete (codec.py:84-85)."""


class BitmapMismatchError(CodecFormatError):
    """Occupancy bitmap popcount disagrees with the payload (codec.py:88-89)."""


class NativeError(RuntimeError):
    """CUDA / NCCL failure inside libfgc_b200."""


def last_error() -> str:
    msg = lib.fgc_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    if status == OK:
        return
    msg = last_error() or what
    if status == ERR_INVALID:
        raise ValueError(msg)
    if status == ERR_NO_CONFIG:
        raise ValueError("eps tuning found no valid configuration")
    if status == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == ERR_HEADER:
        raise CorruptHeaderError(msg)
    if status == ERR_TRUNCATED:
        raise TruncatedPayloadError(msg)
    if status == ERR_BITMAP:
        raise BitmapMismatchError(msg)
    if status == ERR_FORMAT:
        raise CodecFormatError(msg)
    raise NativeError(f"{what}: {msg}" if what else msg)


def kernel_launches() -> int:
    return int(lib.fgc_kernel_launches())
