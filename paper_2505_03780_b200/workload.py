"""Synthetic attention workloads keyed by a ktune ShapeKey dict.

The reference runner allocates inputs from a binding's tensor recipes
(ref/pkg/runner/src/ktune_triton_runner/backends.py:119-137: CPU ``torch.Generator(seed)``, fp32
randn cast to the kernel dtype).  A binding cannot express varlen ``cu_seqlens``, page pools or a
permuted ``block_table`` (ref/pkg/runner/src/ktune_triton_runner/binding.py:154-163), so the attention
runner builds them here from the shape dims (SURVEY §8(d) conventions):

  prefill: {"op":"prefill","batch_size","seq_len" | "seq_len_min","seq_len_max","len_dist",
            "num_q_heads","num_kv_heads","head_dim","causal","dtype","seed"}
  decode:  {"op":"decode","batch_size","seq_len","num_q_heads","num_kv_heads","head_dim",
            "block_size","dtype","seed"[,"kv_dtype":"fp8_e4m3"]}
  fp8 caches hold e4m3(randn * FP8_INV_SCALE) and are read back with k_scale = v_scale =
  1 / FP8_INV_SCALE (per-tensor, vLLM FP8_PER_TENSOR convention).

Small tensors follow the reference exactly (CPU generator, fp32 randn -> bf16).  Tensors above
``CPU_GEN_LIMIT`` elements are drawn from a seeded CUDA generator instead (a 32-GiB paged cache
cannot be drawn on the host per request); ``gen`` forces either.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

CPU_GEN_LIMIT = 1 << 26
FP8_INV_SCALE = 64.0  # randn * 64 stays inside e4m3's +-448 for |x| < 7


def varlen_lengths(shape: dict) -> list[int]:
    B = int(shape["batch_size"])
    if "seq_len" in shape:
        return [int(shape["seq_len"])] * B
    lo, hi = int(shape["seq_len_min"]), int(shape["seq_len_max"])
    dist = shape.get("len_dist", "geometric")
    if B == 1:
        return [hi]
    if dist == "geometric":
        return [int(round(lo * (hi / lo) ** (i / (B - 1)))) for i in range(B)]
    if dist == "linear":
        return [int(round(lo + (hi - lo) * i / (B - 1))) for i in range(B)]
    raise ValueError(f"unknown len_dist {dist!r}")


def _randn(shape, gen_kind: str, seed: int, device, fp8: bool = False) -> torch.Tensor:
    n = 1
    for s in shape:
        n *= int(s)
    kind = gen_kind if gen_kind != "auto" else ("cpu" if n <= CPU_GEN_LIMIT else "cuda")
    dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
    mul = FP8_INV_SCALE if fp8 else 1.0
    if kind == "cpu":
        g = torch.Generator(device="cpu").manual_seed(seed)
        return (torch.randn(shape, generator=g, dtype=torch.float32) * mul).to(dt).to(device)
    g = torch.Generator(device=device).manual_seed(seed)
    out = torch.empty(shape, dtype=dt, device=device)
    # fill in fp32 chunks to bound the temporary
    flat = out.view(-1)
    step = 1 << 27
    for i in range(0, n, step):
        m = min(step, n - i)
        flat[i:i + m] = (torch.randn(m, generator=g, dtype=torch.float32, device=device) * mul).to(dt)
    return out


@dataclass
class PrefillInputs:
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    cu_seqlens: torch.Tensor
    max_seqlen: int
    lens: list
    causal: bool

    @property
    def flops(self) -> int:
        """Algorithmic FLOPs: 4*D*Hq*sum L(L+1)/2 (causal) or 4*D*Hq*sum L^2."""
        D, Hq = self.q.shape[2], self.q.shape[1]
        pairs = sum(L * (L + 1) // 2 if self.causal else L * L for L in self.lens)
        return 4 * D * Hq * pairs


@dataclass
class DecodeInputs:
    q: torch.Tensor
    k_cache: torch.Tensor
    v_cache: torch.Tensor
    block_table: torch.Tensor
    seq_lens: torch.Tensor
    max_seq_len: int
    lens: list
    k_scale: Optional[float] = None
    v_scale: Optional[float] = None

    @property
    def kv_bytes(self) -> int:
        """K+V bytes the decode must read: 2 * sum(n) * Hkv * D * elem (2 for bf16, 1 for fp8)."""
        Hkv, D = self.k_cache.shape[2], self.k_cache.shape[3]
        return 2 * sum(self.lens) * Hkv * D * self.k_cache.element_size()

    @property
    def total_bytes(self) -> int:
        """K+V + Q + O + block_table + seq_lens bytes."""
        return (self.kv_bytes + 2 * self.q.numel() * 2 + self.block_table.numel() * 4 + self.seq_lens.numel() * 4)


def make_prefill(shape: dict, device="cuda", gen: str = "auto", seed: Optional[int] = None) -> PrefillInputs:
    seed = int(shape.get("seed", 0)) if seed is None else seed
    lens = varlen_lengths(shape)
    T = sum(lens)
    Hq, Hkv, D = int(shape["num_q_heads"]), int(shape["num_kv_heads"]), int(shape["head_dim"])
    q = _randn((T, Hq, D), gen, seed, device)
    k = _randn((T, Hkv, D), gen, seed + 1, device)
    v = _randn((T, Hkv, D), gen, seed + 2, device)
    cu = torch.zeros(len(lens) + 1, dtype=torch.int32)
    cu[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int32), 0)
    return PrefillInputs(q, k, v, cu.to(device), max(lens) if lens else 0, lens, bool(shape.get("causal", True)))


def make_decode(shape: dict, device="cuda", gen: str = "auto", seed: Optional[int] = None,
                lens: Optional[list] = None, extra_blocks: int = 0) -> DecodeInputs:
    seed = int(shape.get("seed", 0)) if seed is None else seed
    B = int(shape["batch_size"])
    ctx = int(shape["seq_len"])
    Hq, Hkv, D = int(shape["num_q_heads"]), int(shape["num_kv_heads"]), int(shape["head_dim"])
    bs = int(shape.get("block_size", 16))
    lens = list(lens) if lens is not None else [ctx] * B
    max_blocks = (max(lens) + bs - 1) // bs if lens else 1
    max_blocks = max(max_blocks, 1)
    NB = B * max_blocks + extra_blocks
    q = _randn((B, Hq, D), gen, seed, device)
    fp8 = str(shape.get("kv_dtype", "bfloat16")).startswith(("fp8", "float8"))
    kc = _randn((NB, bs, Hkv, D), gen, seed + 1, device, fp8=fp8)
    vc = _randn((NB, bs, Hkv, D), gen, seed + 2, device, fp8=fp8)
    g = torch.Generator(device="cpu").manual_seed(seed + 3)
    perm = torch.randperm(NB, generator=g)[: B * max_blocks].to(torch.int32).reshape(B, max_blocks)
    sc = 1.0 / FP8_INV_SCALE if fp8 else None
    return DecodeInputs(q, kc, vc, perm.to(device), torch.tensor(lens, dtype=torch.int32, device=device),
                        max(lens) if lens else 0, lens, sc, sc)


# the BASELINE.json configurations
C1 = {"op": "prefill", "batch_size": 1, "seq_len": 512, "num_q_heads": 32, "num_kv_heads": 8, "head_dim": 128,
      "causal": True, "dtype": "bfloat16", "seed": 0}
C2 = {"op": "decode", "batch_size": 64, "seq_len": 4096, "num_q_heads": 32, "num_kv_heads": 8, "head_dim": 128,
      "block_size": 16, "dtype": "bfloat16", "seed": 0}
C3 = {"op": "prefill", "batch_size": 16, "seq_len_min": 128, "seq_len_max": 8192, "len_dist": "geometric",
      "num_q_heads": 32, "num_kv_heads": 8, "head_dim": 128, "causal": True, "dtype": "bfloat16", "seed": 0}
C4 = {"op": "decode", "batch_size": 256, "seq_len": 32768, "num_q_heads": 64, "num_kv_heads": 8, "head_dim": 128,
      "block_size": 16, "dtype": "bfloat16", "seed": 0}


# ----------------------------------------------------------------------------- sharded workloads
# Multi-GPU: the path shards with no exchange step, so each rank builds ONLY its
# shard.  Content is a function of the global unit (sequence for decode, kv head for prefill), never
# of the sharding, so any rank — rank 0 validating a gathered result — can rebuild any unit.
_SEQ_STRIDE = 1_000_003


def _unit_randn(shape, seed: int, unit: int, salt: int, device, fp8: bool = False) -> torch.Tensor:
    g = torch.Generator(device=device).manual_seed(seed * _SEQ_STRIDE + unit * 8 + salt)
    x = torch.randn(shape, generator=g, dtype=torch.float32, device=device)
    return (x * FP8_INV_SCALE).to(torch.float8_e4m3fn) if fp8 else x.to(torch.bfloat16)


def decode_sequence(shape: dict, b: int, device="cuda"):
    """q [Hq, D], k/v [ctx, Hkv, D] of global sequence b of a sharded decode workload."""
    seed = int(shape.get("seed", 0))
    ctx, Hq, Hkv, D = (int(shape[k]) for k in ("seq_len", "num_q_heads", "num_kv_heads", "head_dim"))
    fp8 = str(shape.get("kv_dtype", "bfloat16")).startswith(("fp8", "float8"))
    q = _unit_randn((Hq, D), seed, b, 0, device)
    k = _unit_randn((ctx, Hkv, D), seed, b, 1, device, fp8)
    v = _unit_randn((ctx, Hkv, D), seed, b, 2, device, fp8)
    return q, k, v


def make_decode_shard(shape: dict, start: int, count: int, device="cuda") -> DecodeInputs:
    """Sequences [start, start + count) of the decode workload `shape` (every one seq_len long),
    paged into a pool holding only this shard's pages, block table permuted (seeded by start)."""
    ctx, Hq, Hkv, D = (int(shape[k]) for k in ("seq_len", "num_q_heads", "num_kv_heads", "head_dim"))
    bs = int(shape.get("block_size", 16))
    nblk = (ctx + bs - 1) // bs
    fp8 = str(shape.get("kv_dtype", "bfloat16")).startswith(("fp8", "float8"))
    dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
    NB = max(1, count * nblk)
    kc = torch.zeros((NB, bs, Hkv, D), dtype=dt, device=device)
    vc = torch.zeros_like(kc)
    q = torch.empty((count, Hq, D), dtype=torch.bfloat16, device=device)
    g = torch.Generator(device="cpu").manual_seed(int(shape.get("seed", 0)) * _SEQ_STRIDE + start)
    perm = torch.randperm(NB, generator=g).to(torch.int32)
    bt = perm[: count * nblk].reshape(count, nblk).to(device)
    pad = nblk * bs - ctx
    for i in range(count):
        qi, ki, vi = decode_sequence(shape, start + i, device)
        q[i] = qi
        rows = bt[i].long()
        if pad:
            ki = torch.cat([ki, torch.zeros((pad, Hkv, D), dtype=dt, device=device)])
            vi = torch.cat([vi, torch.zeros((pad, Hkv, D), dtype=dt, device=device)])
        kc[rows] = ki.view(nblk, bs, Hkv, D)
        vc[rows] = vi.view(nblk, bs, Hkv, D)
    sc = 1.0 / FP8_INV_SCALE if fp8 else None
    return DecodeInputs(q, kc, vc, bt, torch.full((count,), ctx, dtype=torch.int32, device=device), ctx,
                        [ctx] * count, sc, sc)


def prefill_kv_head(shape: dict, kvh: int, device="cuda"):
    """q [T, G, D] (the G q heads of kv head kvh), k/v [T, 1, D] of a head-sharded prefill workload."""
    seed = int(shape.get("seed", 0))
    T = sum(varlen_lengths(shape))
    Hq, Hkv, D = int(shape["num_q_heads"]), int(shape["num_kv_heads"]), int(shape["head_dim"])
    G = Hq // Hkv
    return (_unit_randn((T, G, D), seed, kvh, 3, device), _unit_randn((T, 1, D), seed, kvh, 4, device),
            _unit_randn((T, 1, D), seed, kvh, 5, device))


def make_prefill_heads(shape: dict, kv_heads: range, device="cuda") -> PrefillInputs:
    """kv heads `kv_heads` (and their q heads) of the prefill workload `shape`: the head shard a
    rank owns when prefill is split by GQA group."""
    lens = varlen_lengths(shape)
    parts = [prefill_kv_head(shape, h, device) for h in kv_heads]
    q = torch.cat([p[0] for p in parts], 1).contiguous()
    k = torch.cat([p[1] for p in parts], 1).contiguous()
    v = torch.cat([p[2] for p in parts], 1).contiguous()
    cu = torch.zeros(len(lens) + 1, dtype=torch.int32)
    cu[1:] = torch.cumsum(torch.tensor(lens, dtype=torch.int32), 0)
    return PrefillInputs(q, k, v, cu.to(device), max(lens), lens, bool(shape.get("causal", True)))
