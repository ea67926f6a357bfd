"""CPU oracle for the attention hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` legs
import this module, always as the checker (never as the thing measured or shipped).

Two restatements of the same semantics (see oracle/attn_oracle.c header for the citations):
  * ``prefill`` / ``decode``       — ctypes over oracle/_build/liboracle.so (fp64, OpenMP);
  * ``prefill_np`` / ``decode_np`` — numpy fp64, used to cross-check the C one on small cases.
Both take bf16 tensors as ``numpy.uint16`` bit patterns (or torch bf16 tensors) and return
fp64 numpy arrays.  Pinned against tests/golden/*.npz (vLLM 0.22.0 triton_unified_attention
under TRITON_INTERPRET=1; generator: tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "attn_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        i = ctypes.c_int
        lib.oracle_prefill.argtypes = [P, P, P, P, i, i, i, i, i, ctypes.c_double, P, P]
        lib.oracle_prefill.restype = None
        lib.oracle_decode.argtypes = [P, P, P, P, P, i, i, i, i, i, i, ctypes.c_double, P]
        lib.oracle_decode.restype = None
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def num_threads() -> int:
    return int(_load().oracle_num_threads())


def as_bf16_bits(x) -> np.ndarray:
    """torch bf16 tensor (any device) or uint16 array -> contiguous uint16 numpy array."""
    if isinstance(x, np.ndarray):
        assert x.dtype == np.uint16
        return np.ascontiguousarray(x)
    import torch

    assert x.dtype == torch.bfloat16, x.dtype
    return x.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16)


def bf16_bits_to_f64(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _i32(x) -> np.ndarray:
    if not isinstance(x, np.ndarray):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(x, dtype=np.int32)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def prefill(q, k, v, cu_seqlens, causal=True, scale=None, with_lse=False):
    """q [T,Hq,D], k/v [T,Hkv,D] bf16 -> O [T,Hq,D] fp64 (and LSE [Hq,T] natural log)."""
    qb, kb, vb = as_bf16_bits(q), as_bf16_bits(k), as_bf16_bits(v)
    cu = _i32(cu_seqlens)
    T, Hq, D = qb.shape
    Hkv = kb.shape[1]
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = np.zeros((T, Hq, D), dtype=np.float64)
    lse = np.zeros((Hq, T), dtype=np.float64) if with_lse else None
    _load().oracle_prefill(_ptr(qb), _ptr(kb), _ptr(vb), _ptr(cu), len(cu) - 1, Hq, Hkv, D, int(bool(causal)),
                           scale, _ptr(out), _ptr(lse) if lse is not None else None)
    return (out, lse) if with_lse else out


def decode(q, k_cache, v_cache, block_table, seq_lens, scale=None):
    """q [B,Hq,D], caches [NB,bs,Hkv,D] bf16 -> O [B,Hq,D] fp64."""
    qb, kb, vb = as_bf16_bits(q), as_bf16_bits(k_cache), as_bf16_bits(v_cache)
    bt, sl = _i32(block_table), _i32(seq_lens)
    B, Hq, D = qb.shape
    _, bs, Hkv, _ = kb.shape
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = np.zeros((B, Hq, D), dtype=np.float64)
    _load().oracle_decode(_ptr(qb), _ptr(kb), _ptr(vb), _ptr(bt), _ptr(sl), B, Hq, Hkv, D, bs, bt.shape[1], scale,
                          _ptr(out))
    return out


# ----------------------------------------------------------------------------- numpy restatement
def prefill_np(q, k, v, cu_seqlens, causal=True, scale=None):
    qf, kf, vf = (bf16_bits_to_f64(as_bf16_bits(x)) for x in (q, k, v))
    cu = _i32(cu_seqlens)
    T, Hq, D = qf.shape
    G = Hq // kf.shape[1]
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = np.zeros_like(qf)
    for s in range(len(cu) - 1):
        a, b = int(cu[s]), int(cu[s + 1])
        L = b - a
        if L == 0:
            continue
        kk = np.repeat(kf[a:b], G, axis=1)  # [L,Hq,D]
        vv = np.repeat(vf[a:b], G, axis=1)
        sc = np.einsum("ihd,jhd->hij", qf[a:b], kk) * scale
        if causal:
            sc = np.where(np.tril(np.ones((L, L), dtype=bool))[None], sc, -np.inf)
        sc = sc - sc.max(-1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(-1, keepdims=True)
        out[a:b] = np.einsum("hij,jhd->ihd", p, vv)
    return out


def prefill_blas(q, k, v, cu_seqlens, causal=True, scale=None, heads=None, chunk=1024):
    """Same semantics as ``prefill`` in fp64 through BLAS matmuls (torch fp64 on the host cores:
    multithreaded matmuls AND elementwise passes), chunked over query rows so a causal chunk only
    touches keys up to its last row: the full-size parity tests (all of C3's 16 sequences x 32
    heads) finish in seconds instead of minutes.  ``heads`` restricts the work (and the output)
    to those q heads.  Returns fp64 numpy [T, len(heads), D]."""
    import torch

    qf, kf, vf = (torch.from_numpy(bf16_bits_to_f64(as_bf16_bits(x))) for x in (q, k, v))
    cu = _i32(cu_seqlens)
    T, Hq, D = qf.shape
    G = Hq // kf.shape[1]
    heads = list(range(Hq)) if heads is None else list(heads)
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = torch.zeros((T, len(heads), D), dtype=torch.float64)
    for s in range(len(cu) - 1):
        a, b = int(cu[s]), int(cu[s + 1])
        for hi, h in enumerate(heads):
            kk, vv = kf[a:b, h // G], vf[a:b, h // G]  # [L, D]
            for r0 in range(0, b - a, chunk):
                r1 = min(b - a, r0 + chunk)
                kend = r1 if causal else b - a
                sc = (qf[a + r0:a + r1, h] @ kk[:kend].T) * scale  # [rows, kend]
                if causal:
                    mask = torch.arange(kend)[None, :] > torch.arange(r0, r1)[:, None]
                    sc.masked_fill_(mask, -float("inf"))
                sc -= sc.amax(-1, keepdim=True)
                sc.exp_()
                out[a + r0:a + r1, hi] = (sc @ vv[:kend]) / sc.sum(-1, keepdim=True)
    return out.numpy()


def decode_np(q, k_cache, v_cache, block_table, seq_lens, scale=None):
    qf = bf16_bits_to_f64(as_bf16_bits(q))
    kc, vc = (bf16_bits_to_f64(as_bf16_bits(x)) for x in (k_cache, v_cache))
    bt, sl = _i32(block_table), _i32(seq_lens)
    B, Hq, D = qf.shape
    bs, Hkv = kc.shape[1], kc.shape[2]
    G = Hq // Hkv
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = np.zeros_like(qf)
    for b in range(B):
        n = int(sl[b])
        if n == 0:
            continue
        t = np.arange(n)
        pages = bt[b, t // bs]
        kk = np.repeat(kc[pages, t % bs], G, axis=1)  # [n,Hq,D]
        vv = np.repeat(vc[pages, t % bs], G, axis=1)
        sc = np.einsum("hd,nhd->hn", qf[b], kk) * scale
        sc -= sc.max(-1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(-1, keepdims=True)
        out[b] = np.einsum("hn,nhd->hd", p, vv)
    return out


# ----------------------------------------------------------------------------- fp8 (e4m3) KV cache
def e4m3_table() -> np.ndarray:
    """All 256 OCP FP8 E4M3 (``e4m3fn``) byte values as fp64: bias 7, no infinities, S.1111.111 = NaN,
    exponent 0 = subnormal 2^-6 * m/8 (OCP 8-bit floating point specification v1.0, Table 1)."""
    b = np.arange(256)
    s = np.where(b >> 7, -1.0, 1.0)
    e = (b >> 3) & 15
    m = (b & 7).astype(np.float64)
    v = np.where(e == 0, 2.0 ** -6 * m / 8, 2.0 ** (e - 7.0) * (1 + m / 8))
    v = s * v
    v[(e == 15) & ((b & 7) == 7)] = np.nan
    return v


_E4M3 = None


def as_u8(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        assert x.dtype == np.uint8
        return np.ascontiguousarray(x)
    import torch

    return x.detach().cpu().contiguous().view(torch.uint8).numpy()


def decode_fp8_np(q, k_cache, v_cache, block_table, seq_lens, k_scale, v_scale, scale=None):
    """Paged decode over an e4m3 cache: K = e4m3(k_cache) * k_scale, V = e4m3(v_cache) * v_scale
    (vLLM FP8_PER_TENSOR: vllm/v1/attention/ops/triton_unified_attention.py _cast_kv_tile), the rest
    exactly as ``decode_np``.  q bf16, caches uint8 [NB,bs,Hkv,D] -> O fp64 [B,Hq,D]."""
    global _E4M3
    if _E4M3 is None:
        _E4M3 = e4m3_table()
    qf = bf16_bits_to_f64(as_bf16_bits(q))
    kc, vc = as_u8(k_cache), as_u8(v_cache)
    bt, sl = _i32(block_table), _i32(seq_lens)
    B, Hq, D = qf.shape
    bs, Hkv = kc.shape[1], kc.shape[2]
    G = Hq // Hkv
    scale = float(scale) if scale else 1.0 / np.sqrt(D)
    out = np.zeros_like(qf)
    for b in range(B):
        n = int(sl[b])
        if n == 0:
            continue
        t = np.arange(n)
        pages = bt[b, t // bs]
        kk = np.repeat(_E4M3[kc[pages, t % bs]] * float(k_scale), G, axis=1)  # [n,Hq,D]
        vv = np.repeat(_E4M3[vc[pages, t % bs]] * float(v_scale), G, axis=1)
        sc = np.einsum("hd,nhd->hn", qf[b], kk) * scale
        sc -= sc.max(-1, keepdims=True)
        p = np.exp(sc)
        p /= p.sum(-1, keepdims=True)
        out[b] = np.einsum("hn,nhd->hd", p, vv)
    return out


def quantize_e4m3_np(x: np.ndarray, inv_scale: float) -> np.ndarray:
    """fp64 -> e4m3 bytes, round-to-nearest-even on the value grid, saturating at +-448 (the
    ``cvt.rn.satfinite.e4m3x2.f32`` semantics the cache-append kernel uses)."""
    global _E4M3
    if _E4M3 is None:
        _E4M3 = e4m3_table()
    y = np.clip(np.asarray(x, dtype=np.float64) * inv_scale, -448.0, 448.0)
    pos = np.arange(0, 127)  # non-negative finite codes, ascending values
    grid = _E4M3[pos]
    mag = np.abs(y)
    i = np.clip(np.searchsorted(grid, mag), 1, len(grid) - 1)
    lo, hi = grid[i - 1], grid[i]
    pick_hi = (mag - lo > hi - mag) | ((mag - lo == hi - mag) & (pos[i] % 2 == 0))
    code = np.where(pick_hi, pos[i], pos[i - 1])
    code = np.where(mag <= grid[0], 0, code)
    return (code | np.where(np.signbit(y), 0x80, 0)).astype(np.uint8)  # -tiny -> -0, like cvt.rn


if __name__ == "__main__":  # pragma: no cover
    print(build(force=bool(os.environ.get("FORCE"))))
