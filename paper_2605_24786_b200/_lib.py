"""ctypes binding of `libconfkv_b200.so` (the C ABI in include/confkv_b200.h).

There is no CPU fallback: importing the engine without the built library or
without a CUDA device raises. Status codes map to the reference's exception
types (config.py:16 ConfigError, ValueError, RuntimeError).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from .config import ConfigError

LIB_PATH = Path(__file__).resolve().parent / "libconfkv_b200.so"

CKV_OK, CKV_EINVAL, CKV_ECONFIG, CKV_ERUNTIME, CKV_ECUDA, CKV_ENOMEM = 0, -1, -2, -3, -4, -5
DTYPE_F32, DTYPE_BF16, DTYPE_F64 = 0, 1, 2

# device-side status bits (ckv_internal.cuh StatusBits)
ST_NONFINITE, ST_NOATTEND, ST_OVERFLOW, ST_SEGOVERFLOW, ST_SCHEDULE, ST_SHAPE = 1, 2, 4, 8, 32, 64
POLICY_CONFKV, POLICY_FULL, POLICY_SLIDING, POLICY_HEAVY_HITTER = 0, 1, 2, 3
POLICY_MATCHED_RANDOM, POLICY_MATCHED_RECENCY, POLICY_MATCHED_ATTENTION = 4, 5, 6


class CkvConfig(C.Structure):
    _fields_ = [
        ("tau", C.c_double),
        ("n_high", C.c_int32), ("n_low", C.c_int32), ("protected_p", C.c_int32),
        ("fp16_window_w", C.c_int32), ("block_size_b", C.c_int32),
        ("alpha", C.c_double), ("ema_lambda", C.c_double),
        ("w_entropy", C.c_double), ("w_margin", C.c_double), ("w_top", C.c_double),
        ("quantize", C.c_int32), ("temperature_mode", C.c_int32),
        ("temperature", C.c_double),
        ("policy", C.c_int32), ("policy_param", C.c_int32),
    ]


class CkvShape(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("num_layers", "num_heads", "num_kv_heads", "head_dim", "vocab_size")]


class CkvLayerRecord(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("len_pre", "len_post", "evicted", "int8_count", "len_after", "num_segments", "status", "int8_codes")]


class CkvSeqRecord(C.Structure):
    _fields_ = [("score", C.c_double), ("entropy_norm", C.c_double), ("margin", C.c_double),
                ("margin_sig", C.c_double), ("top_prob", C.c_double),
                ("tier_high", C.c_int32), ("token", C.c_int32), ("status", C.c_int32), ("pad", C.c_int32)]


P = C.c_void_p
I32, I64 = C.c_int32, C.c_int64

_SIGS = {
    "ckv_last_error": (C.c_char_p, []),
    "ckv_version": (C.c_int, []),
    "ckv_create": (C.c_int, [C.POINTER(CkvConfig), C.POINTER(CkvShape), I32, I32, I32, P, C.POINTER(P)]),
    "ckv_destroy": (C.c_int, [P]),
    "ckv_reset": (C.c_int, [P, P]),
    "ckv_device_bytes": (I64, [P]),
    "ckv_launch_count": (I64, [P]),
    "ckv_begin_prefill": (C.c_int, [P, I32]),
    "ckv_prefill": (C.c_int, [P, I32, I32, P, P, I32, I32, P]),
    "ckv_attend": (C.c_int, [P, I32, I32, P, P, P, P]),
    "ckv_attend_fork": (C.c_int, [P, I32, I32, P, P, P, P, P]),
    "ckv_attend_conf": (C.c_int, [P, I32, I32, P, P, P, P, I32, I64, P, P]),
    "ckv_stage_rows": (C.c_int, [P, I32, P, I32, P]),
    "ckv_confidence": (C.c_int, [P, P, I32, I64, P]),
    "ckv_stage_weights": (C.c_int, [P, I32, I32, P, I32, P]),
    "ckv_head_partial": (C.c_int, [P, I32, I32, P, P, P, P]),
    "ckv_stage_mass": (C.c_int, [P, I32, I32, P, I32, P]),
    "ckv_confidence_partial": (C.c_int, [P, P, I32, I64, I64, P, P]),
    "ckv_confidence_merge": (C.c_int, [P, P, I32, I64, P]),
    "ckv_manage": (C.c_int, [P, I32, P, P, P, P, P]),
    "ckv_step": (C.c_int, [P, I32, P, I32, I64, P, P, P, P, P, P, P]),
    "ckv_tokens": (C.c_int, [P, P, P]),
    "ckv_pipe_submit": (C.c_int, [P, P, P, P, P, P, I64, P, P, P, I32, P, P, I64, P, P, I64]),
    "ckv_pack_outputs": (C.c_int, [P, P, P, I32, P]),
    "ckv_set_victims": (C.c_int, [P, P, P, I32, P]),
    "ckv_victims_out": (C.c_int, [P, P]),
    "ckv_qkv_split": (C.c_int, [P, I32, I32, I32, P, P, P, P]),
    "ckv_read_records": (C.c_int, [P, P, P, P]),
    "ckv_copy_records": (C.c_int, [P, P, P, P]),
    "ckv_read_cache": (C.c_int, [P, I32, I32, P, P] + [P] * 12 + [P]),
    "ckv_read_staged": (C.c_int, [P, I32, I32, I32, P, P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    # CKV_LIB: load another build of the same ABI (A/B kernel experiments under tools/)
    p = Path(path) if path else Path(os.environ.get("CKV_LIB", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"{p} not built: run `python -m paper_2605_24786_b200.build` "
            "(the B200 path has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == CKV_OK:
        return
    msg = load().ckv_last_error().decode(errors="replace")
    if status == CKV_ECONFIG:
        raise ConfigError(msg)
    if status == CKV_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)
