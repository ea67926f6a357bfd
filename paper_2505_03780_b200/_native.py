"""ctypes binding of libb200attn.so (include/b200attn.h).

The product path has exactly one implementation: the sm_100a kernels in this library.  If the
library is missing or cannot be loaded this module raises — there is no CPU / eager fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("B200ATTN_LIB", PKG_DIR / "_lib" / "libb200attn.so"))

OK = 0
UNSUPPORTED_CONFIG = 1
SMEM_OVERFLOW = 2
TMEM_OVERFLOW = 3
BAD_ARGS = 4
CUDA_ERROR = 5
INVALID_CODES = (UNSUPPORTED_CONFIG, SMEM_OVERFLOW, TMEM_OVERFLOW)

_P = ctypes.c_void_p
_I = ctypes.c_int32


class PrefillVariant(ctypes.Structure):
    _fields_ = [("block_m", _I), ("block_n", _I), ("num_warps", _I), ("num_stages", _I), ("waves_per_eu", _I),
                ("pre_load_v", _I)]


class PrefillParams(ctypes.Structure):
    _fields_ = [("q", _P), ("k", _P), ("v", _P), ("o", _P), ("cu_seqlens", _P), ("lse", _P), ("num_seqs", _I),
                ("total_tokens", _I), ("max_seqlen", _I), ("num_q_heads", _I), ("num_kv_heads", _I),
                ("head_dim", _I), ("causal", _I), ("softmax_scale", ctypes.c_float), ("workspace", _P),
                ("workspace_bytes", ctypes.c_size_t)]


class DecodeVariant(ctypes.Structure):
    _fields_ = [("num_splits", _I), ("num_stages", _I), ("tile_n", _I)]


class DecodeParams(ctypes.Structure):
    _fields_ = [("q", _P), ("k_cache", _P), ("v_cache", _P), ("block_table", _P), ("seq_lens", _P), ("o", _P),
                ("workspace", _P), ("workspace_bytes", ctypes.c_size_t), ("batch", _I), ("num_q_heads", _I),
                ("num_kv_heads", _I), ("head_dim", _I), ("block_size", _I), ("num_blocks", _I),
                ("max_blocks_per_seq", _I), ("max_seq_len", _I), ("softmax_scale", ctypes.c_float),
                ("kv_dtype", _I), ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float)]


ABI_VERSION = 2
KV_BF16 = 0
KV_FP8_E4M3 = 1


class B200AttnError(RuntimeError):
    """A non-OK status from the C ABI.  ``invalid`` is True for config rejections."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.status_name = STATUS_NAMES.get(status, "unknown")
        self.invalid = status in INVALID_CODES
        super().__init__(f"{self.status_name}: {message}")


STATUS_NAMES = {OK: "ok", UNSUPPORTED_CONFIG: "unsupported_config", SMEM_OVERFLOW: "smem_overflow",
                TMEM_OVERFLOW: "tmem_overflow", BAD_ARGS: "bad_args", CUDA_ERROR: "cuda_error"}

# every symbol include/b200attn.h declares (tests check the library exports all of them)
EXPORTS = (
    "b200attn_abi_version", "b200attn_build_info", "b200attn_status_string", "b200attn_last_error",
    "b200attn_prefill_supported", "b200attn_decode_supported", "b200attn_prefill_workspace_size", "b200attn_prefill",
    "b200attn_decode_workspace_size", "b200attn_decode_num_splits", "b200attn_decode_launches", "b200attn_decode",
    "b200attn_decode_partial",
    "b200attn_combine",
    "b200attn_cache_append", "b200attn_cache_append_fp8", "b200attn_selftest_umma",
    "b200attn_decode_ingest", "b200attn_mapped_ptr",
)

_lib = None


def load():
    """Load (once) and type the native library; raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"native library {LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no non-CUDA fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    PP, PV, DP, DV = (ctypes.POINTER(t) for t in (PrefillParams, PrefillVariant, DecodeParams, DecodeVariant))
    lib.b200attn_abi_version.restype = ctypes.c_int
    lib.b200attn_build_info.restype = ctypes.c_char_p
    lib.b200attn_status_string.restype = ctypes.c_char_p
    lib.b200attn_status_string.argtypes = [ctypes.c_int]
    lib.b200attn_last_error.restype = ctypes.c_char_p
    lib.b200attn_prefill_supported.argtypes = [PP, PV, ctypes.c_char_p, ctypes.c_size_t]
    lib.b200attn_decode_supported.argtypes = [DP, DV, ctypes.c_char_p, ctypes.c_size_t]
    lib.b200attn_prefill.argtypes = [PP, PV, _P]
    lib.b200attn_prefill_workspace_size.argtypes = [PP]
    lib.b200attn_prefill_workspace_size.restype = ctypes.c_size_t
    lib.b200attn_decode.argtypes = [DP, DV, _P]
    lib.b200attn_decode_partial.argtypes = [DP, DV, _P]
    lib.b200attn_decode_workspace_size.argtypes = [DP, DV]
    lib.b200attn_decode_workspace_size.restype = ctypes.c_size_t
    lib.b200attn_decode_num_splits.argtypes = [DP, DV]
    lib.b200attn_decode_launches.argtypes = [DP, DV]
    lib.b200attn_combine.argtypes = [_P, _P, _P, _I, _I, _P]
    lib.b200attn_cache_append.argtypes = [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P]
    lib.b200attn_cache_append_fp8.argtypes = [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, ctypes.c_float,
                                              ctypes.c_float, _P]
    lib.b200attn_selftest_umma.argtypes = [ctypes.c_int, _P, _P, _P, _P]
    lib.b200attn_decode_ingest.argtypes = [_P, _P, ctypes.c_int64, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I,
                                           ctypes.c_float, ctypes.c_float, _P]
    lib.b200attn_mapped_ptr.argtypes = [_P, ctypes.POINTER(ctypes.c_void_p)]
    for name in ("b200attn_prefill_supported", "b200attn_decode_supported", "b200attn_prefill", "b200attn_decode",
                 "b200attn_decode_partial",
                 "b200attn_combine", "b200attn_cache_append", "b200attn_cache_append_fp8", "b200attn_selftest_umma",
                 "b200attn_decode_num_splits", "b200attn_decode_launches", "b200attn_decode_ingest",
                 "b200attn_mapped_ptr"):
        getattr(lib, name).restype = ctypes.c_int
    if lib.b200attn_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libb200attn ABI {lib.b200attn_abi_version()} != {ABI_VERSION}; rebuild the library")
    _lib = lib
    return lib


def check(status: int):
    if status != OK:
        raise B200AttnError(status, load().b200attn_last_error().decode(errors="replace"))


def reason_buffer():
    return ctypes.create_string_buffer(512)
