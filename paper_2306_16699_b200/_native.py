"""ctypes binding of the C ABI (include/rinr_b200.h) exported by the in-tree
``_lib/librinr_b200.so``.  There is no fallback: if the library is missing the
import fails loudly (build it with ``python -m paper_2306_16699_b200.build``)."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .errors import raise_for_status

# RINR_LIB_PATH selects another build of the same ABI (tools/checked_build.sh's
# bounds-asserting library); the default is the in-tree product build
LIB_PATH = Path(os.environ.get("RINR_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "librinr_b200.so")

# enums (include/rinr_b200.h)
OUT_F32, OUT_BF16, OUT_U8 = 0, 1, 2
LAYOUT_NCHW, LAYOUT_NHWC = 0, 1
PREC_FP32, PREC_BF16, PREC_EXACT = 0, 1, 2
SIN_MUFU, SIN_ACCURATE = 0, 1
AUG_NONE, AUG_OFFSET, AUG_CROP = 0, 1, 2
FLAG_OVERLAP_PROLOGUE = 1
FLAG_PREFETCH_NEXT = 2

EXPORTS = (
    "rinr_abi_version", "rinr_last_error", "rinr_last_error_record", "rinr_archive_validate", "rinr_archive_shard",
    "rinr_store_create", "rinr_store_destroy", "rinr_store_info", "rinr_store_record_meta",
    "rinr_dequantize", "rinr_decode", "rinr_prune_l1", "rinr_quantize", "rinr_psnr", "rinr_fit", "rinr_fit_render",
    "rinr_serialize_size", "rinr_serialize_write",
)


class StoreInfo(C.Structure):
    _fields_ = [
        ("num_records", C.c_int64), ("total_records", C.c_int64),
        ("shard_rank", C.c_uint32), ("shard_world", C.c_uint32),
        ("device", C.c_int32), ("uniform_arch", C.c_int32), ("n_dims", C.c_int32),
        ("dims", C.c_uint16 * 32), ("omega", C.c_double),
        ("max_param_count", C.c_int64), ("max_record_bytes", C.c_int64), ("device_bytes", C.c_int64),
        ("uniform_source", C.c_int32), ("source_h", C.c_uint32), ("source_w", C.c_uint32),
    ]


class FitParams(C.Structure):  # rinr_fit_params_t (include/rinr_b200_encoder.h)
    _fields_ = [("h", C.c_int32), ("w", C.c_int32), ("steps", C.c_int32), ("sin_mode", C.c_int32),
                ("lr0", C.c_double), ("omega", C.c_double), ("curve_cap", C.c_int32), ("sched", C.c_void_p)]


class SerializeArgs(C.Structure):  # rinr_serialize_args_t (include/rinr_b200_writer.h)
    _fields_ = [
        ("dims", C.POINTER(C.c_int32)), ("n_layers", C.c_int), ("n", C.c_int64),
        ("source_h", C.c_uint32), ("source_w", C.c_uint32), ("omega", C.c_double), ("quant_bits", C.c_int),
        ("d_w", C.c_void_p), ("d_mask", C.c_void_p), ("d_b", C.c_void_p), ("d_scale", C.c_void_p),
        ("d_zp", C.c_void_p), ("d_const", C.c_void_p), ("d_codes", C.c_void_p),
        ("id_prefix", C.c_char_p), ("first_id", C.c_int64), ("id_width", C.c_int),
    ]


class DecodeParams(C.Structure):
    _fields_ = [
        ("out_h", C.c_int32), ("out_w", C.c_int32), ("out_dtype", C.c_int32), ("out_layout", C.c_int32),
        ("precision", C.c_int32), ("sin_mode", C.c_int32), ("aug_mode", C.c_int32),
        ("mean", C.c_float * 3), ("std", C.c_float * 3), ("flags", C.c_int32),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2306_16699_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32p = C.c_void_p, C.c_int64, C.POINTER(C.c_int32)
    L.rinr_abi_version.restype = C.c_int
    L.rinr_last_error.restype = C.c_char_p
    L.rinr_last_error_record.restype = i64
    L.rinr_archive_validate.argtypes = [vp, C.c_size_t, C.POINTER(i64)]
    L.rinr_archive_shard.argtypes = [vp, C.c_size_t, C.c_uint32, C.c_uint32, vp, i64, C.POINTER(i64)]
    L.rinr_store_create.argtypes = [vp, C.c_size_t, C.c_int, C.c_uint32, C.c_uint32, C.POINTER(vp)]
    L.rinr_store_destroy.argtypes = [vp]
    L.rinr_store_info.argtypes = [vp, C.POINTER(StoreInfo)]
    L.rinr_store_record_meta.argtypes = [vp, i64, C.POINTER(i64), C.c_char_p, C.c_size_t,
                                         C.POINTER(C.c_size_t), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    L.rinr_dequantize.argtypes = [vp, vp, i64, vp, i64, vp, vp]
    L.rinr_decode.argtypes = [vp, vp, i64, C.POINTER(DecodeParams), vp, vp, vp, vp]
    L.rinr_prune_l1.argtypes = [vp, C.c_int, i64, vp, vp, vp, C.c_int, vp, vp]
    L.rinr_quantize.argtypes = [vp, C.c_int, i64, C.c_int, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.rinr_psnr.argtypes = [vp, vp, i64, i64, C.c_int, vp, vp, vp]
    L.rinr_fit.argtypes = [vp, C.c_int, i64, vp, vp, vp, vp, C.POINTER(FitParams), vp, vp, vp, vp, vp, vp]
    L.rinr_fit_render.argtypes = [vp, C.c_int, i64, vp, vp, C.c_int32, C.c_int32, C.c_double, C.c_int32, vp, vp]
    L.rinr_serialize_size.argtypes = [C.POINTER(SerializeArgs), vp, vp, vp, vp]
    L.rinr_serialize_write.argtypes = [C.POINTER(SerializeArgs), vp, vp, vp, vp, vp, vp]
    L.rinr_diag_launch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, C.POINTER(C.c_double)]
    L.rinr_diag_launch.restype = C.c_int
    for name in EXPORTS:
        if name != "rinr_abi_version" and name not in ("rinr_last_error", "rinr_last_error_record"):
            getattr(L, name).restype = C.c_int
    if L.rinr_abi_version() != 1:
        raise ImportError("librinr_b200.so ABI version mismatch")
    _lib = L
    return L


def check(code: int) -> None:
    if code != 0:
        L = lib()
        raise_for_status(code, L.rinr_last_error().decode("utf-8", "replace"), int(L.rinr_last_error_record()))


def archive_validate(data: bytes) -> int:
    """Host-only validation of an archive image; returns the record count."""
    n = C.c_int64(0)
    arr = host_view(data)
    check(lib().rinr_archive_validate(arr.ctypes.data if arr.size else None, arr.size, C.byref(n)))
    return n.value


def archive_shard(data, rank: int, world: int):
    """Global indices of the records a Store(rank, world) keeps (host-only)."""
    import numpy as np  # noqa: PLC0415
    arr = host_view(data)
    cnt = C.c_int64(0)
    ptr = arr.ctypes.data if arr.size else None
    check(lib().rinr_archive_shard(ptr, arr.size, rank, world, None, 0, C.byref(cnt)))
    out = np.zeros(cnt.value, np.int64)
    check(lib().rinr_archive_shard(ptr, arr.size, rank, world, out.ctypes.data if out.size else None, out.size,
                                   C.byref(cnt)))
    return out


def host_view(data):
    """Zero-copy uint8 view of bytes / bytearray / memoryview / numpy data."""
    import numpy as np  # noqa: PLC0415
    if isinstance(data, np.ndarray):
        return np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    return np.frombuffer(data, dtype=np.uint8)
