"""Public attention entry points: ``prefill_varlen``, ``paged_decode``, ``cache_append``.

These are the framework's drop-in for the kernel call the reference runner makes for one
(config, shape) — ``self.kernel[grid](*args, **kwargs)`` (ref/pkg/runner/src/ktune_triton_runner/
backends.py:164-165) — with ``config`` keyed by the autotuner space's parameter names exactly as
``KernelBinding.kernel_kwargs`` produces them (ref/pkg/runner/src/ktune_triton_runner/binding.py:146-147;
space: ref/pkg/src/ktune/fixtures/flash_attention.space.json:3-16).  Layouts follow the paper's
kernel family as upstreamed in vLLM: q/k/v ``[tokens, heads, 128]``, paged caches
``[num_blocks, block_size, kv_heads, 128]``.

Every call goes to libb200attn.so (sm_100a tcgen05/TMA kernels).  torch is used only for device
memory and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import itertools
import math
from typing import Mapping, Optional

import torch

from . import _native
from .dispatch import default_decode_config, default_prefill_config

PREFILL_PARAMS = ("BLOCK_M", "BLOCK_N", "num_warps", "num_stages", "waves_per_eu", "PRE_LOAD_V")
DECODE_PARAMS = ("num_splits", "num_stages", "TILE_N")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _check(t: torch.Tensor, name: str, dtype=torch.bfloat16, ndim=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")


def prefill_variant(config: Mapping) -> _native.PrefillVariant:
    missing = [p for p in PREFILL_PARAMS if p not in config]
    if missing:
        raise KeyError(f"config is missing space parameter {missing[0]!r}")
    return _native.PrefillVariant(int(config["BLOCK_M"]), int(config["BLOCK_N"]), int(config["num_warps"]),
                                  int(config["num_stages"]), int(config["waves_per_eu"]),
                                  int(bool(config["PRE_LOAD_V"])))


def decode_variant(config: Mapping) -> _native.DecodeVariant:
    missing = [p for p in DECODE_PARAMS if p not in config]
    if missing:
        raise KeyError(f"config is missing space parameter {missing[0]!r}")
    return _native.DecodeVariant(int(config["num_splits"]), int(config["num_stages"]), int(config["TILE_N"]))


def _prefill_params(q, k, v, out, cu_seqlens, max_seqlen, softmax_scale, causal, lse):
    T, Hq, D = q.shape
    return _native.PrefillParams(
        _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(cu_seqlens), _ptr(lse), cu_seqlens.numel() - 1, T,
        int(max_seqlen), Hq, k.shape[1], D, int(bool(causal)), float(softmax_scale or 0.0))


def prefill_supported(q_shape, kv_heads, num_seqs, max_seqlen, config: Mapping, causal=True):
    """(ok, reason) for a config on a shape, without launching."""
    lib = _native.load()
    T, Hq, D = q_shape
    p = _native.PrefillParams(None, None, None, None, None, None, num_seqs, T, max_seqlen, Hq, kv_heads, D,
                              int(causal), 0.0, None, 0)
    buf = _native.reason_buffer()
    rc = lib.b200attn_prefill_supported(p, prefill_variant(config), buf, len(buf))
    return rc, buf.value.decode()


def prefill_varlen(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, cu_seqlens: torch.Tensor, max_seqlen: int,
                   out: Optional[torch.Tensor] = None, softmax_scale: Optional[float] = None, causal: bool = True,
                   config: Optional[Mapping] = None, return_lse: bool = False):
    """Causal varlen prefill: q [T,Hq,128], k/v [T,Hkv,128] bf16, cu_seqlens [B+1] int32 (device).

    ``config`` is a flash_attention.space.json point (BLOCK_M, BLOCK_N, num_warps, num_stages,
    waves_per_eu, PRE_LOAD_V); default: the per-shape dispatch table.
    """
    lib = _native.load()
    _check_prefill_shapes(q, k, v, cu_seqlens, out)
    with _on(q.device):
        if out is None:
            out = torch.empty_like(q)
        lse = torch.empty(q.shape[1], q.shape[0], device=q.device, dtype=torch.float32) if return_lse else None
        if config is None:
            config = default_prefill_config(num_seqs=cu_seqlens.numel() - 1, total_tokens=q.shape[0],
                                            max_seqlen=int(max_seqlen), num_q_heads=q.shape[1],
                                            num_kv_heads=k.shape[1], head_dim=q.shape[2], causal=causal)
        p = _prefill_params(q, k, v, out, cu_seqlens, max_seqlen, softmax_scale, causal, lse)
        stream = torch.cuda.current_stream(q.device)
        ws = _workspace(q.device, lib.b200attn_prefill_workspace_size(p), kind="prefill", stream=stream)
        p.workspace, p.workspace_bytes = ws.data_ptr(), ws.numel()
        _native.check(lib.b200attn_prefill(p, prefill_variant(config), stream.cuda_stream))
    return (out, lse) if return_lse else out


def _same_device(*ts):
    dev = ts[0].device
    for t in ts[1:]:
        if t is not None and t.device != dev:
            raise ValueError(f"all tensors must be on {dev}, got one on {t.device}")


def _check_prefill_shapes(q, k, v, cu_seqlens, out=None):
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _check(t, n, ndim=3)
    _check(cu_seqlens, "cu_seqlens", dtype=torch.int32, ndim=1)
    if k.shape != v.shape or k.shape[0] != q.shape[0] or k.shape[2] != q.shape[2]:
        raise ValueError(f"shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    if k.shape[1] == 0 or q.shape[1] % k.shape[1]:
        raise ValueError(f"num_q_heads={q.shape[1]} is not a multiple of num_kv_heads={k.shape[1]}")
    if cu_seqlens.numel() < 2:
        raise ValueError("cu_seqlens needs at least 2 entries (one sequence)")
    if out is not None:
        _check(out, "out", ndim=3)
        if out.shape != q.shape:
            raise ValueError(f"out{tuple(out.shape)} must match q{tuple(q.shape)}")
    _same_device(q, k, v, cu_seqlens, out)


_workspaces: "OrderedDict" = None
_WS_MAX = 32  # bound: streams come and go in a server; least recently used buffers are dropped


def _workspace(device, nbytes: int, kind: str = "decode", stream=None) -> Optional[torch.Tensor]:
    """Scratch for one launch, cached per (device, stream, kind).

    The prefill buffer carries the self-resetting work counter and the decode buffer the split
    partials that the combine pass reads, so two launches in flight on different streams must not
    share one (include/b200attn.h: launches are stream-ordered and reentrant).  Launches on ONE
    stream are ordered, so they can."""
    global _workspaces
    if nbytes == 0:
        return None
    if _workspaces is None:
        from collections import OrderedDict

        _workspaces = OrderedDict()
    s = stream if stream is not None else torch.cuda.current_stream(device)
    key = (device.type, device.index, s.cuda_stream, kind)
    buf = _workspaces.get(key)
    if buf is None or buf.numel() < nbytes:
        # zeroed: the prefill work counter must start at 0 (the kernel's last CTA re-zeroes it);
        # allocated on the stream that uses it, so the caching allocator never hands it to another
        with torch.cuda.stream(s):
            buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _workspaces[key] = buf
    _workspaces.move_to_end(key)
    while len(_workspaces) > _WS_MAX:
        _workspaces.popitem(last=False)
    return buf


FP8_DTYPE = torch.float8_e4m3fn  # OCP e4m3 KV cache (vLLM FP8_PER_TENSOR semantics)


def _kv_dtype_code(cache: torch.Tensor) -> int:
    if cache.dtype == torch.bfloat16:
        return _native.KV_BF16
    if cache.dtype == FP8_DTYPE:
        return _native.KV_FP8_E4M3
    raise TypeError(f"KV cache must be bfloat16 or float8_e4m3fn, got {cache.dtype}")


def _check_cache(t: torch.Tensor, name: str):
    _check(t, name, dtype=t.dtype if t.dtype in (torch.bfloat16, FP8_DTYPE) else torch.bfloat16, ndim=4)


def _decode_params(q, k_cache, v_cache, block_table, seq_lens, out, max_seq_len, softmax_scale, ws=None, ws_bytes=0,
                   k_scale=None, v_scale=None):
    B, Hq, D = q.shape
    NB, bs, Hkv, _ = k_cache.shape
    return _native.DecodeParams(
        _ptr(q), _ptr(k_cache), _ptr(v_cache), _ptr(block_table), _ptr(seq_lens), _ptr(out), _ptr(ws), ws_bytes, B,
        Hq, Hkv, D, bs, NB, block_table.shape[1], int(max_seq_len), float(softmax_scale or 0.0),
        _kv_dtype_code(k_cache), float(k_scale or 1.0), float(v_scale or 1.0))


def decode_supported(q_shape, cache_shape, max_blocks_per_seq, max_seq_len, config: Mapping, kv_dtype="bfloat16"):
    lib = _native.load()
    B, Hq, D = q_shape
    NB, bs, Hkv, _ = cache_shape
    code = _native.KV_FP8_E4M3 if str(kv_dtype).startswith(("fp8", "float8")) else _native.KV_BF16
    p = _native.DecodeParams(None, None, None, None, None, None, None, 0, B, Hq, Hkv, D, bs, NB, max_blocks_per_seq,
                             max_seq_len, 0.0, code, 1.0, 1.0)
    buf = _native.reason_buffer()
    rc = lib.b200attn_decode_supported(p, decode_variant(config), buf, len(buf))
    return rc, buf.value.decode()


def _decode_config(q, k_cache, block_table, max_seq_len) -> dict:
    """The dispatch table's config for this shape; a flat (TILE_N = 16) pick whose smem does not fit
    (very large batches keep a per-sequence prefix in smem) drops to the deepest ring that fits, else
    to the split kernel."""
    kv = _kv_name(k_cache)
    cfg = default_decode_config(batch_size=q.shape[0], seq_len=int(max_seq_len), num_q_heads=q.shape[1],
                                num_kv_heads=k_cache.shape[2], head_dim=q.shape[2], block_size=k_cache.shape[1],
                                kv_dtype=kv)
    if int(cfg["TILE_N"]) != 16 or q.shape[0] <= 1024:
        return cfg
    for ns in range(int(cfg["num_stages"]), 1, -1):
        c = dict(cfg, num_stages=ns)
        if decode_supported(tuple(q.shape), tuple(k_cache.shape), block_table.shape[1], int(max_seq_len), c, kv)[0] == 0:
            return c
    return dict(num_splits=0, num_stages=4, TILE_N=128)


def paged_decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_table: torch.Tensor,
                 seq_lens: torch.Tensor, max_seq_len: Optional[int] = None, out: Optional[torch.Tensor] = None,
                 softmax_scale: Optional[float] = None, config: Optional[Mapping] = None,
                 k_scale: Optional[float] = None, v_scale: Optional[float] = None):
    """Paged-KV decode: q [B,Hq,128]; caches [NB,bs,Hkv,128] bf16 or float8_e4m3fn (then K = k_cache * k_scale,
    V = v_cache * v_scale, per-tensor); block_table [B,maxblk] int32; seq_lens [B] int32.
    ``max_seq_len`` (host int) sizes the split grid; defaults to the block-table capacity so no
    device->host sync is needed.
    """
    lib = _native.load()
    _check_decode_shapes(q, k_cache, v_cache, block_table, seq_lens, out)
    if max_seq_len is None:
        max_seq_len = block_table.shape[1] * k_cache.shape[1]
    with _on(q.device):
        if out is None:
            out = torch.empty_like(q)
        if config is None:
            config = _decode_config(q, k_cache, block_table, max_seq_len)
        var = decode_variant(config)
        p = _decode_params(q, k_cache, v_cache, block_table, seq_lens, out, max_seq_len, softmax_scale,
                           k_scale=k_scale, v_scale=v_scale)
        nbytes = lib.b200attn_decode_workspace_size(p, var)
        stream = torch.cuda.current_stream(q.device)
        ws = _workspace(q.device, nbytes, kind="decode", stream=stream)
        if ws is not None:
            p.workspace = ws.data_ptr()
            p.workspace_bytes = ws.numel()
        _native.check(lib.b200attn_decode(p, var, stream.cuda_stream))
    return out


def _check_decode_shapes(q, k_cache, v_cache, block_table, seq_lens, out=None):
    """Cross-tensor checks: a mismatch here would otherwise be an out-of-bounds device access."""
    _check(q, "q", ndim=3)
    _check_cache(k_cache, "k_cache")
    _check_cache(v_cache, "v_cache")
    if k_cache.dtype != v_cache.dtype:
        raise TypeError("k_cache / v_cache dtype mismatch")
    if k_cache.shape != v_cache.shape:
        raise ValueError("k_cache / v_cache shape mismatch")
    _check(block_table, "block_table", dtype=torch.int32, ndim=2)
    _check(seq_lens, "seq_lens", dtype=torch.int32, ndim=1)
    B, Hq, D = q.shape
    if k_cache.shape[3] != D:
        raise ValueError(f"cache head_dim {k_cache.shape[3]} != q head_dim {D}")
    Hkv = k_cache.shape[2]
    if Hkv == 0 or Hq % Hkv:
        raise ValueError(f"num_q_heads={Hq} is not a multiple of num_kv_heads={Hkv}")
    if block_table.shape[0] != B or seq_lens.numel() != B:
        raise ValueError(f"batch mismatch: q {B}, block_table {block_table.shape[0]}, seq_lens {seq_lens.numel()}")
    if out is not None:
        _check(out, "out", ndim=3)
        if out.shape != q.shape:
            raise ValueError(f"out{tuple(out.shape)} must match q{tuple(q.shape)}")
    _same_device(q, k_cache, v_cache, block_table, seq_lens, out)


def decode_num_splits(q_shape, cache_shape, max_blocks_per_seq, max_seq_len, config: Mapping) -> int:
    lib = _native.load()
    B, Hq, D = q_shape
    NB, bs, Hkv, _ = cache_shape
    p = _native.DecodeParams(None, None, None, None, None, None, None, 0, B, Hq, Hkv, D, bs, NB, max_blocks_per_seq,
                             max_seq_len, 0.0, _native.KV_BF16, 1.0, 1.0)
    return int(lib.b200attn_decode_num_splits(p, decode_variant(config)))


def combine(part_o: torch.Tensor, part_ml: torch.Tensor, out: torch.Tensor):
    """K3 alone: part_o [rows, S, 128] fp32, part_ml [rows, S, 2] (max in log2 units, sum) -> out [rows,128]."""
    lib = _native.load()
    _check(part_o, "part_o", dtype=torch.float32, ndim=3)
    _check(part_ml, "part_ml", dtype=torch.float32, ndim=3)
    _check(out, "out")
    rows, S, _ = part_o.shape
    _native.check(lib.b200attn_combine(_ptr(part_o), _ptr(part_ml), _ptr(out), rows, S,
                                       torch.cuda.current_stream(out.device).cuda_stream))
    return out


def _kv_name(cache: torch.Tensor) -> str:
    return "fp8_e4m3" if cache.dtype == FP8_DTYPE else "bfloat16"


def cache_append(new_k: torch.Tensor, new_v: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor,
                 slot_mapping: torch.Tensor, k_scale: Optional[float] = None, v_scale: Optional[float] = None):
    """Write new_k/new_v [N, Hkv, 128] bf16 into pages: slot = page * block_size + offset (int64, < 0
    skips).  float8_e4m3fn caches store satfinite_rn(x / k_scale) (resp. v_scale)."""
    lib = _native.load()
    _check(new_k, "new_k", ndim=3)
    _check(new_v, "new_v", ndim=3)
    _check_cache(k_cache, "k_cache")
    _check_cache(v_cache, "v_cache")
    _check(slot_mapping, "slot_mapping", dtype=torch.int64, ndim=1)
    NB, bs, Hkv, D = k_cache.shape
    if k_cache.shape != v_cache.shape:
        raise ValueError("k_cache / v_cache shape mismatch")
    if new_k.shape != new_v.shape or new_k.shape[1:] != (Hkv, D):
        raise ValueError(f"new_k{tuple(new_k.shape)} / new_v{tuple(new_v.shape)} must be [N, {Hkv}, {D}]")
    if slot_mapping.numel() != new_k.shape[0]:
        raise ValueError(f"slot_mapping has {slot_mapping.numel()} entries for {new_k.shape[0]} tokens")
    _same_device(new_k, new_v, k_cache, v_cache, slot_mapping)
    if k_cache.dtype != v_cache.dtype:
        raise TypeError("k_cache / v_cache dtype mismatch")
    with _on(new_k.device):
        stream = torch.cuda.current_stream(new_k.device).cuda_stream
        if _kv_dtype_code(k_cache) == _native.KV_FP8_E4M3:
            _native.check(lib.b200attn_cache_append_fp8(_ptr(new_k), _ptr(new_v), _ptr(k_cache), _ptr(v_cache),
                                                        _ptr(slot_mapping), new_k.shape[0], Hkv, D, bs, NB,
                                                        float(k_scale or 1.0), float(v_scale or 1.0), stream))
            return
        _native.check(lib.b200attn_cache_append(_ptr(new_k), _ptr(new_v), _ptr(k_cache), _ptr(v_cache),
                                                _ptr(slot_mapping), new_k.shape[0], Hkv, D, bs, NB, stream))


class _NoGuard:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


_NO_GUARD = _NoGuard()


def _on(device):
    """Make `device` current for a launch (kernels go to the current device; the stream passed
    belongs to `device`).  Free when it already is current — the common single-GPU case."""
    if torch.cuda.current_device() == device.index:
        return _NO_GUARD
    return torch.cuda.device(device)


def selftest_umma(mode: int, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """tcgen05 descriptor self-test (see include/b200attn.h)."""
    lib = _native.load()
    d = torch.empty((128, 16 if mode == 2 else 128), device=a.device, dtype=torch.float32)
    _native.check(lib.b200attn_selftest_umma(mode, _ptr(a), _ptr(b), _ptr(d),
                                             torch.cuda.current_stream(a.device).cuda_stream))
    return d


def default_scale(head_dim: int) -> float:
    return 1.0 / math.sqrt(head_dim)


class DecodePlan:
    """Plan/run split for serving loops and CUDA-graph capture: validates once, pins the
    params struct and workspace, then ``run()`` is a single C-ABI call (K2 [+K3])."""

    def __init__(self, q, k_cache, v_cache, block_table, seq_lens, out=None, max_seq_len=None, config=None,
                 softmax_scale=None, k_scale=None, v_scale=None):
        self.lib = _native.load()
        _check_decode_shapes(q, k_cache, v_cache, block_table, seq_lens, out)
        self.max_seq_len = int(max_seq_len if max_seq_len is not None else block_table.shape[1] * k_cache.shape[1])
        self.out = torch.empty_like(q) if out is None else out
        self.config = dict(config or _decode_config(q, k_cache, block_table, self.max_seq_len))
        self.var = decode_variant(self.config)
        self.p = _decode_params(q, k_cache, v_cache, block_table, seq_lens, self.out, self.max_seq_len, softmax_scale,
                                k_scale=k_scale, v_scale=v_scale)
        nbytes = self.lib.b200attn_decode_workspace_size(self.p, self.var)
        # zeroed: the flat kernel's per-sequence arrival counters must start at 0 (they self-reset)
        self.ws = torch.zeros(max(nbytes, 1), dtype=torch.uint8, device=q.device) if nbytes else None
        if self.ws is not None:
            self.p.workspace, self.p.workspace_bytes = self.ws.data_ptr(), self.ws.numel()
        self.num_splits = int(self.lib.b200attn_decode_num_splits(self.p, self.var))
        self.device = q.device
        # the params struct holds raw pointers: keep the tensors alive as long as the plan
        self._tensors = (q, k_cache, v_cache, block_table, seq_lens, self.out)

    def kernels_per_run(self) -> int:
        return int(self.lib.b200attn_decode_launches(self.p, self.var))

    def run(self, stream=None):
        with _on(self.device):
            s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
            _native.check(self.lib.b200attn_decode(self.p, self.var, s))
        return self.out

    def run_partial(self, stream=None):
        """K2 only (the dominant kernel), for roofline timing."""
        with _on(self.device):
            s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
            _native.check(self.lib.b200attn_decode_partial(self.p, self.var, s))


class PrefillPlan:
    def __init__(self, q, k, v, cu_seqlens, max_seqlen, out=None, causal=True, config=None, softmax_scale=None):
        self.lib = _native.load()
        _check_prefill_shapes(q, k, v, cu_seqlens, out)
        self.out = torch.empty_like(q) if out is None else out
        self.config = dict(config or default_prefill_config(
            num_seqs=cu_seqlens.numel() - 1, total_tokens=q.shape[0], max_seqlen=int(max_seqlen),
            num_q_heads=q.shape[1], num_kv_heads=k.shape[1], head_dim=q.shape[2], causal=causal))
        self.var = prefill_variant(self.config)
        self.p = _prefill_params(q, k, v, self.out, cu_seqlens, max_seqlen, softmax_scale, causal, None)
        self.ws = torch.zeros(max(1, self.lib.b200attn_prefill_workspace_size(self.p)), dtype=torch.uint8,
                              device=q.device)
        self.p.workspace, self.p.workspace_bytes = self.ws.data_ptr(), self.ws.numel()
        self.device = q.device
        self._tensors = (q, k, v, cu_seqlens, self.out)  # raw pointers in self.p: keep them alive

    def run(self, stream=None):
        with _on(self.device):
            s = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
            _native.check(self.lib.b200attn_prefill(self.p, self.var, s))
        return self.out


def pack_pinned(tensors, align: int = 256):
    """Copy host tensors into one pinned byte buffer; returns (buffer, [(offset, shape, dtype)])."""
    offs, n = [], 0
    for t in tensors:
        n = (n + align - 1) // align * align
        offs.append(n)
        n += t.numel() * t.element_size()
    buf = torch.empty(max(n, 1), dtype=torch.uint8).pin_memory()
    views = []
    for t, o in zip(tensors, offs):
        nb = t.numel() * t.element_size()
        buf[o:o + nb].copy_(t.contiguous().view(-1).view(torch.uint8))
        views.append((o, tuple(t.shape), t.dtype))
    return buf, views


def unpack_view(buf: torch.Tensor, v) -> torch.Tensor:
    o, shape, dtype = v
    nb = math.prod(shape) * torch.empty(0, dtype=dtype).element_size()
    return buf[o:o + nb].view(dtype).view(shape)


class DecodeStep:
    """One serving decode step as ONE CUDA graph, host buffers in and out:

        H2D (pinned staging: q, the new token's K/V, slot_mapping, seq_lens)
        -> cache_append (new K/V into its page slot) -> paged_decode -> D2H (output, pinned)

    With one chunk (the default) the step is three kernels and no copy nodes (``zero_copy``): one
    ingest kernel reads q, seq_lens and the new K/V straight from the pinned staging buffer over
    PCIe (device-mapped host memory), copying q/seq_lens to HBM and appending K/V into the pages in
    the same launch, then K2' + K3' run and write the output rows straight into the pinned
    ``out_host`` — the copy-engine nodes, their graph edges and the separate append launch are gone.

    The batch is cut into ``chunks`` contiguous groups of sequences whose transfers overlap the
    other groups' kernels on separate copy streams: H2D(i+1) runs under decode(i) and D2H(i) under
    decode(i+1), so only the first group's inputs and the last group's output sit on the critical
    path.  The graph is: copy stream H2D_i -> event -> compute stream append_i, decode_i -> event ->
    copy stream D2H_i, joined back at the end.

    Inputs are written through ``set_inputs`` (or the per-chunk host views ``chunk_views(i)``);
    ``out_host`` [B, Hq, D] holds the result once the stream reaches the end of the step
    (``sync=True`` waits for it).  The paged KV pool and the block table stay resident on the
    device: a serving loop appends one page index per sequence every ``block_size`` steps, in place."""

    def __init__(self, k_cache, v_cache, block_table, batch: int, num_q_heads: int, max_seq_len=None, config=None,
                 softmax_scale=None, k_scale=None, v_scale=None, chunks: int = 0, zero_copy: bool = True):
        dev = k_cache.device
        _check_cache(k_cache, "k_cache")
        Hkv, D = k_cache.shape[2], k_cache.shape[3]
        B, Hq = int(batch), int(num_q_heads)
        if chunks <= 0:
            # one chunk: a decode launch per chunk costs more (ramp + tail) than the copies it hides
            # (C2: 217 us at 1 chunk vs 233 / 262 / 239 us at 2 / 3 / 4, r2d perf.py e2e)
            chunks = 1
        chunks = max(1, min(chunks, B))
        bounds = [B * i // chunks for i in range(chunks + 1)]
        self.bounds = bounds
        self.chunks = chunks
        # chunk-major pinned staging: chunk i = [q | seq_lens | new_k | new_v | slots] of its rows (q and
        # seq_lens first: the one range the decode kernels read from HBM); views in the order
        # (q, new_k, new_v, slots, seq_lens)
        protos, self._views = [], []
        for i in range(chunks):
            n = bounds[i + 1] - bounds[i]
            protos += [torch.empty(n, Hq, D, dtype=torch.bfloat16), torch.zeros(n, dtype=torch.int32),
                       torch.empty(n, Hkv, D, dtype=torch.bfloat16), torch.empty(n, Hkv, D, dtype=torch.bfloat16),
                       torch.full((n,), -1, dtype=torch.int64)]
        self.stage_h, packed = pack_pinned(protos)
        views = []
        for i in range(chunks):
            q_, sl_, k_, v_, s_ = packed[5 * i:5 * i + 5]
            views += [q_, k_, v_, s_, sl_]
        self.stage_d = torch.empty_like(self.stage_h, device=dev)
        self.out_host = torch.empty(B, Hq, D, dtype=torch.bfloat16).pin_memory()
        self.out_d = torch.empty(B, Hq, D, dtype=torch.bfloat16, device=dev)
        self.h2d_bytes = sum(math.prod(v[1]) * torch.empty(0, dtype=v[2]).element_size() for v in views)
        self.d2h_bytes = self.out_host.numel() * 2
        self.device = dev
        self.plans, ranges = [], []
        for i in range(chunks):
            hv = [unpack_view(self.stage_h, v) for v in views[5 * i:5 * i + 5]]
            dv = [unpack_view(self.stage_d, v) for v in views[5 * i:5 * i + 5]]
            self._views.append(hv)
            lo = packed[5 * i][0]
            last = packed[5 * i + 4]
            hi = last[0] + math.prod(last[1]) * 8  # slots (int64) end the chunk
            ranges.append((lo, hi))
            b0, b1 = bounds[i], bounds[i + 1]
            self.plans.append((DecodePlan(dv[0], k_cache, v_cache, block_table[b0:b1], dv[4], out=self.out_d[b0:b1],
                                          max_seq_len=max_seq_len, config=config, softmax_scale=softmax_scale,
                                          k_scale=k_scale, v_scale=v_scale), dv))
        self.config = self.plans[0][0].config
        self.zero_copy = bool(zero_copy) and chunks == 1
        if self.zero_copy:
            lib = _native.load()

            def mapped(t):
                ptr = ctypes.c_void_p()
                _native.check(lib.b200attn_mapped_ptr(t.data_ptr(), ctypes.byref(ptr)))
                return ptr.value

            plan, dv = self.plans[0]
            plan.p.o = mapped(self.out_host)  # K2' / K3' store the output rows into pinned host memory
            plan._tensors += (self.out_host,)
            sl = packed[1]
            copy_bytes = (sl[0] + math.prod(sl[1]) * 4 + 15) // 16 * 16  # q + seq_lens
            base = mapped(self.stage_h)
            off = {name: packed[j][0] for j, name in ((2, "k"), (3, "v"), (4, "s"))}
            kv_fp8 = _kv_dtype_code(k_cache) == _native.KV_FP8_E4M3
            self._ingest = (base, self.stage_d.data_ptr(), copy_bytes, base + off["k"], base + off["v"],
                            base + off["s"], k_cache.data_ptr(), v_cache.data_ptr(), B, Hkv, D, k_cache.shape[1],
                            k_cache.shape[0], _native.KV_FP8_E4M3 if kv_fp8 else _native.KV_BF16,
                            float(k_scale or 1.0) if kv_fp8 else 1.0, float(v_scale or 1.0) if kv_fp8 else 1.0)
            self._kv = (k_cache, v_cache)

        def body():
            main = torch.cuda.current_stream(dev)
            if self.zero_copy:  # ingest kernel (PCIe reads) -> K2' [+ K3'] (output rows written to host)
                _native.check(_native.load().b200attn_decode_ingest(*self._ingest, main.cuda_stream))
                self.plans[0][0].run()
                return
            if chunks == 1:  # one stream: H2D -> append -> decode -> D2H, no cross-stream edges
                lo, hi = ranges[0]
                plan, dv = self.plans[0]
                self.stage_d[lo:hi].copy_(self.stage_h[lo:hi], non_blocking=True)
                cache_append(dv[1], dv[2], k_cache, v_cache, dv[3], k_scale=k_scale, v_scale=v_scale)
                plan.run()
                self.out_host.copy_(self.out_d, non_blocking=True)
                return
            ev_in = [torch.cuda.Event() for _ in range(chunks)]
            ev_dec = [torch.cuda.Event() for _ in range(chunks)]
            self._cin.wait_stream(main)
            self._cout.wait_stream(main)
            with torch.cuda.stream(self._cin):
                for i, (lo, hi) in enumerate(ranges):
                    self.stage_d[lo:hi].copy_(self.stage_h[lo:hi], non_blocking=True)
                    ev_in[i].record()
            for i, (plan, dv) in enumerate(self.plans):
                main.wait_event(ev_in[i])
                cache_append(dv[1], dv[2], k_cache, v_cache, dv[3], k_scale=k_scale, v_scale=v_scale)
                plan.run()
                ev_dec[i].record(main)
            with torch.cuda.stream(self._cout):
                for i in range(chunks):
                    self._cout.wait_event(ev_dec[i])
                    b0, b1 = bounds[i], bounds[i + 1]
                    self.out_host[b0:b1].copy_(self.out_d[b0:b1], non_blocking=True)
            main.wait_stream(self._cin)
            main.wait_stream(self._cout)

        with _on(dev):
            self._cin, self._cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                body()  # warm: attributes, descriptor prefetch (slots are -1: nothing written)
            torch.cuda.current_stream(dev).wait_stream(s)
            torch.cuda.synchronize(dev)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                body()
        self.done = torch.cuda.Event()

    def chunk_views(self, i: int):
        """host views (q, new_k, new_v, slot_mapping, seq_lens) of chunk i's rows in the staging buffer."""
        return self._views[i]

    def set_inputs(self, q=None, new_k=None, new_v=None, slot_mapping=None, seq_lens=None):
        """Scatter full-batch host tensors into the chunk-major pinned staging buffer."""
        for i in range(self.chunks):
            b0, b1 = self.bounds[i], self.bounds[i + 1]
            for dst, src in zip(self._views[i], (q, new_k, new_v, slot_mapping, seq_lens)):
                if src is not None:
                    dst.copy_(src[b0:b1])

    def __call__(self, sync: bool = False) -> torch.Tensor:
        with _on(self.device):
            self.graph.replay()
            if sync:
                self.done.record()
                self.done.synchronize()
        return self.out_host


class PrefillStep:
    """One serving prefill step as ONE CUDA graph, host buffers in and out:

        H2D (pinned staging: q, k, v, cu_seqlens of a group of sequences) -> prefill_varlen -> D2H

    The varlen batch (``seq_lens``, fixed at construction like a plan) is cut into ``chunks``
    contiguous groups of sequences with about equal token counts.  Group i's H2D runs on one copy
    stream while group i-1 is computed, and group i-1's output is read back on a second copy stream
    while later groups compute or upload — the host links' two directions run at once, so a step
    costs about max(inputs, outputs) / PCIe rate instead of their sum plus the kernels.

    ``set_inputs(q, k, v)`` scatters packed host tensors [tokens, heads, D] into the staging buffer;
    ``out_host`` [tokens, Hq, D] holds the result once the stream reaches the end of the step."""

    def __init__(self, seq_lens, num_q_heads: int, num_kv_heads: int, head_dim: int = 128, causal: bool = True,
                 config=None, softmax_scale=None, chunks: int = 0, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        lens = [int(n) for n in seq_lens]
        T, Hq, Hkv, D = sum(lens), int(num_q_heads), int(num_kv_heads), int(head_dim)
        if chunks <= 0:
            # the copies dominate (C3: 410 MB in, 274 MB out; 7.4 ms of upload at 55 GB/s): with the
            # heaviest group first, 16 groups leave only the lightest group's prefill + read-back after
            # the last upload (C3 step: 8.69 ms at 16 groups, 8.93 at 8, 9.73 at 4; 9.52 at 16 in batch
            # order, whose last group was the 8192-token sequence — perf.py pfe2e, r2p1/r2p2)
            chunks = 16
        chunks = max(1, min(chunks, len(lens)))
        # group boundaries (sequence indices) at ~equal token counts
        bounds, acc, cut = [0], 0, 1
        for i, n in enumerate(lens):
            acc += n
            if cut < chunks and acc >= T * cut / chunks and i + 1 < len(lens):
                bounds.append(i + 1)
                cut += 1
        bounds.append(len(lens))
        self.bounds = bounds
        self.chunks = len(bounds) - 1
        protos, tok = [], [0]
        for i in range(self.chunks):
            g = lens[bounds[i]:bounds[i + 1]]
            n = sum(g)
            tok.append(tok[-1] + n)
            cu = torch.tensor([0] + list(itertools.accumulate(g)), dtype=torch.int32)
            protos += [torch.empty(n, Hq, D, dtype=torch.bfloat16), torch.empty(n, Hkv, D, dtype=torch.bfloat16),
                       torch.empty(n, Hkv, D, dtype=torch.bfloat16), cu]
        self.tok = tok
        self.stage_h, views = pack_pinned(protos)
        self.stage_d = torch.empty_like(self.stage_h, device=dev)
        self.out_host = torch.empty(T, Hq, D, dtype=torch.bfloat16).pin_memory()
        self.out_d = torch.empty(T, Hq, D, dtype=torch.bfloat16, device=dev)
        self.h2d_bytes = self.stage_h.numel()
        self.d2h_bytes = self.out_host.numel() * 2
        self.device = dev
        self._views, self.plans, ranges = [], [], []
        for i in range(self.chunks):
            hv = [unpack_view(self.stage_h, v) for v in views[4 * i:4 * i + 4]]
            dv = [unpack_view(self.stage_d, v) for v in views[4 * i:4 * i + 4]]
            self._views.append(hv)
            lo = views[4 * i][0]
            last = views[4 * i + 3]
            ranges.append((lo, last[0] + math.prod(last[1]) * 4))
            g = lens[bounds[i]:bounds[i + 1]]
            self.plans.append(PrefillPlan(dv[0], dv[1], dv[2], dv[3], max(g), out=self.out_d[tok[i]:tok[i + 1]],
                                          causal=causal, config=config, softmax_scale=softmax_scale))
        self.config = self.plans[0].config
        # groups run heaviest first (causal work ~ sum L^2): what is left after the last upload is
        # that group's prefill + read-back, so it should be the lightest one.  In batch order C3's
        # last group is its 8192-token sequence (~0.5 ms of prefill + 67 MB of read-back).
        self.order = sorted(range(self.chunks), key=lambda i: -sum(n * n for n in lens[bounds[i]:bounds[i + 1]]))
        order = self.order

        def body():
            main = torch.cuda.current_stream(dev)
            ev_in = [torch.cuda.Event() for _ in range(self.chunks)]
            ev_done = [torch.cuda.Event() for _ in range(self.chunks)]
            self._cin.wait_stream(main)
            self._cout.wait_stream(main)
            with torch.cuda.stream(self._cin):
                for i in order:
                    lo, hi = ranges[i]
                    self.stage_d[lo:hi].copy_(self.stage_h[lo:hi], non_blocking=True)
                    ev_in[i].record()
            for i in order:
                main.wait_event(ev_in[i])
                self.plans[i].run()
                ev_done[i].record(main)
            with torch.cuda.stream(self._cout):
                for i in order:
                    self._cout.wait_event(ev_done[i])
                    self.out_host[tok[i]:tok[i + 1]].copy_(self.out_d[tok[i]:tok[i + 1]], non_blocking=True)
            main.wait_stream(self._cin)
            main.wait_stream(self._cout)

        with _on(dev):
            self._cin, self._cout = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                body()  # warm: attributes, tensor maps, schedule workspaces
            torch.cuda.current_stream(dev).wait_stream(s)
            torch.cuda.synchronize(dev)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                body()
        self.done = torch.cuda.Event()

    def set_inputs(self, q=None, k=None, v=None):
        """Scatter packed host tensors [tokens, heads, D] into the group-major pinned staging buffer."""
        for i in range(self.chunks):
            t0, t1 = self.tok[i], self.tok[i + 1]
            for dst, src in zip(self._views[i][:3], (q, k, v)):
                if src is not None:
                    dst.copy_(src[t0:t1])

    def __call__(self, sync: bool = False) -> torch.Tensor:
        with _on(self.device):
            self.graph.replay()
            if sync:
                self.done.record()
                self.done.synchronize()
        return self.out_host
