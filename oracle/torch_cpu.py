"""PyTorch-native CPU attention — TEST / BASELINE INFRASTRUCTURE ONLY (like the rest of oracle/).

The paper normalises its kernels to "the PyTorch-native implementation" (ref/PAPER.md:20-21).
This is that implementation on the host: torch ``scaled_dot_product_attention`` on all host cores
(in fp32, or in bf16 — torch's CPU flash kernel, fp32 accumulation), from the same bf16 inputs,
with the same semantics as oracle/attn_oracle.c (GQA h -> h/G, causal varlen via cu_seqlens,
paged gather via block_table).  It is the fast CPU
variant next to the fp64 oracle in bench.py's ``cpu_baseline`` and ``--impl reference`` legs
(BASELINE.md §4); tests/test_oracle.py pins it to the fp64 oracle.  Only tests/ and bench.py's CPU
legs call it, and never on the product path.
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.nn.functional as F


def set_threads(n: int | None = None) -> int:
    n = n or os.cpu_count() or 1
    torch.set_num_threads(n)
    return torch.get_num_threads()


def prefill(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, cu_seqlens, causal: bool = True,
            scale: float | None = None, dtype=torch.float32) -> torch.Tensor:
    """q [T,Hq,D], k/v [T,Hkv,D] (bf16, CPU) -> fp32 [T,Hq,D]; one SDPA call per sequence, computed
    in `dtype` (fp32, or bf16 = torch's CPU flash kernel with fp32 accumulation, AMX on this host)."""
    cu = [int(x) for x in (cu_seqlens.tolist() if hasattr(cu_seqlens, "tolist") else cu_seqlens)]
    Hq, Hkv = q.shape[1], k.shape[1]
    out = torch.empty(q.shape, dtype=torch.float32)
    for s in range(len(cu) - 1):
        a, b = cu[s], cu[s + 1]
        if b == a:
            continue
        qq = q[a:b].to(dtype).transpose(0, 1)[None]
        kk = k[a:b].to(dtype).transpose(0, 1)[None]
        vv = v[a:b].to(dtype).transpose(0, 1)[None]
        o = F.scaled_dot_product_attention(qq, kk, vv, is_causal=causal, scale=scale, enable_gqa=Hq != Hkv)
        out[a:b] = o[0].transpose(0, 1)
    return out


def decode(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_table, seq_lens,
           scale: float | None = None, dtype=torch.float32) -> torch.Tensor:
    """q [B,Hq,D] bf16, caches [NB,bs,Hkv,D] bf16, block_table [B,maxblk], seq_lens [B] -> fp32 [B,Hq,D]."""
    B, Hq, D = q.shape
    bs, Hkv = k_cache.shape[1], k_cache.shape[2]
    bt = block_table.long()
    out = torch.zeros(B, Hq, D, dtype=torch.float32)
    for b in range(B):
        n = int(seq_lens[b])
        if n == 0:
            continue
        nblk = (n + bs - 1) // bs
        pages = bt[b, :nblk]
        kk = k_cache[pages].reshape(nblk * bs, Hkv, D)[:n].to(dtype).transpose(0, 1)[None]
        vv = v_cache[pages].reshape(nblk * bs, Hkv, D)[:n].to(dtype).transpose(0, 1)[None]
        qq = q[b].to(dtype)[None, :, None]
        out[b] = F.scaled_dot_product_attention(qq, kk, vv, scale=scale, enable_gqa=Hq != Hkv)[0, :, 0]
    return out


def to_np(x: torch.Tensor) -> np.ndarray:
    return x.double().numpy()
