"""Generate the golden attention vectors that pin oracle/attn_oracle.c.

Run HERE (the build container), not on the GPU box:  python tests/golden/make_golden.py

Source of truth: the reference has no attention arithmetic (ref/SPEC.md:16, :605); the paper's
kernel is the IBM Triton flash-attention family (ref/PAPER.md:108-110), upstreamed into vLLM as
``vllm/v1/attention/ops/triton_unified_attention.py::unified_attention`` (third-party, vLLM 0.22.0
as installed in this image).  That kernel is executed with ``TRITON_INTERPRET=1`` on the CPU
(numpy-backed Triton interpreter).  The interpreter mishandles bf16 storage, so bf16-valued
inputs are passed in fp32 storage (exact) and the kernel runs its dots in fp32; outputs are
stored as fp32.  Each fixture holds the bf16 input bit patterns and the kernel's output.

Prefill goldens place K/V in a paged cache with a permuted block table and call the kernel with
q_len == k_len per sequence (causal), exactly the varlen-prefill semantics; decode goldens use
q_len == 1 per sequence.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ["TRITON_INTERPRET"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402

OUT = Path(__file__).resolve().parent


def bf16_inputs(shape, gen):
    x = torch.randn(shape, generator=gen, dtype=torch.float32).to(torch.bfloat16)
    return x


def bits(x: torch.Tensor) -> np.ndarray:
    return x.contiguous().view(torch.int16).numpy().view(np.uint16)


def run_unified(q, kc, vc, cu_q, seqused, max_q, max_k, bt, scale):
    from vllm.v1.attention.ops.triton_unified_attention import unified_attention

    out = torch.zeros_like(q)
    unified_attention(q, kc, vc, out, cu_q, max_q, seqused, max_k, scale, True, (-1, -1), bt, 0, None, None, None)
    return out


def page(k: torch.Tensor, lens, bs, gen):
    """contiguous [T,H,D] per-sequence K -> paged cache [NB,bs,H,D] + block table."""
    H, D = k.shape[1], k.shape[2]
    nblk = [(L + bs - 1) // bs for L in lens]
    NB = sum(nblk) + 2
    perm = torch.randperm(NB, generator=gen)
    cache = torch.zeros(NB, bs, H, D, dtype=k.dtype)
    bt = torch.zeros(len(lens), max(nblk), dtype=torch.int32)
    off, pi = 0, 0
    for s, L in enumerate(lens):
        for j in range(nblk[s]):
            p = int(perm[pi])
            pi += 1
            bt[s, j] = p
            n = min(bs, L - j * bs)
            cache[p, :n] = k[off + j * bs: off + j * bs + n]
        off += L
    return cache, bt, perm


def prefill_case(name, lens, Hq, Hkv, D=128, bs=16, seed=0):
    g = torch.Generator().manual_seed(seed)
    T = sum(lens)
    q, k, v = bf16_inputs((T, Hq, D), g), bf16_inputs((T, Hkv, D), g), bf16_inputs((T, Hkv, D), g)
    gp = torch.Generator().manual_seed(seed + 100)
    kc, bt, perm = page(k, lens, bs, gp)
    gp = torch.Generator().manual_seed(seed + 100)
    vc, bt2, _ = page(v, lens, bs, gp)
    assert torch.equal(bt, bt2)
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    out = run_unified(q.float(), kc.float(), vc.float(), cu, torch.tensor(lens, dtype=torch.int32), max(lens),
                      max(lens), bt, D ** -0.5)
    np.savez_compressed(OUT / f"{name}.npz", kind="prefill", q=bits(q), k=bits(k), v=bits(v), cu_seqlens=cu.numpy(),
                        out=out.numpy().astype(np.float32), source="vllm-0.22.0 triton_unified_attention "
                        "(TRITON_INTERPRET=1, fp32 storage of bf16 inputs)")
    print(name, "T", T, "out|max|", float(out.abs().max()))


def decode_case(name, lens, Hq, Hkv, D=128, bs=16, seed=0):
    g = torch.Generator().manual_seed(seed)
    B = len(lens)
    nblk = [(L + bs - 1) // bs for L in lens]
    NB = sum(nblk) + 3
    q = bf16_inputs((B, Hq, D), g)
    kc, vc = bf16_inputs((NB, bs, Hkv, D), g), bf16_inputs((NB, bs, Hkv, D), g)
    perm = torch.randperm(NB, generator=g)
    bt = torch.zeros(B, max(nblk), dtype=torch.int32)
    pi = 0
    for b in range(B):
        for j in range(nblk[b]):
            bt[b, j] = int(perm[pi])
            pi += 1
    cu = torch.arange(B + 1, dtype=torch.int32)
    sl = torch.tensor(lens, dtype=torch.int32)
    out = run_unified(q.float(), kc.float(), vc.float(), cu, sl, 1, max(lens), bt, D ** -0.5)
    np.savez_compressed(OUT / f"{name}.npz", kind="decode", q=bits(q), k_cache=bits(kc), v_cache=bits(vc),
                        block_table=bt.numpy(), seq_lens=sl.numpy(), out=out.numpy().astype(np.float32),
                        source="vllm-0.22.0 triton_unified_attention (TRITON_INTERPRET=1, fp32 storage of "
                        "bf16 inputs)")
    print(name, "B", B, "out|max|", float(out.abs().max()))


def decode_fp8_case(name, lens, Hq, Hkv, D=128, bs=16, seed=0, k_scale=1 / 64, v_scale=1 / 32):
    """fp8 e4m3 paged cache, per-tensor descales (vLLM KVQuantMode.FP8_PER_TENSOR)."""
    from vllm.v1.attention.ops.triton_unified_attention import KVQuantMode, unified_attention

    g = torch.Generator().manual_seed(seed)
    B = len(lens)
    nblk = [(L + bs - 1) // bs for L in lens]
    NB = sum(nblk) + 3
    q = bf16_inputs((B, Hq, D), g)
    kc = (torch.randn((NB, bs, Hkv, D), generator=g) / k_scale).to(torch.float8_e4m3fn)
    vc = (torch.randn((NB, bs, Hkv, D), generator=g) / v_scale).clamp(-448, 448).to(torch.float8_e4m3fn)
    perm = torch.randperm(NB, generator=g)
    bt = torch.zeros(B, max(nblk), dtype=torch.int32)
    pi = 0
    for b in range(B):
        for j in range(nblk[b]):
            bt[b, j] = int(perm[pi])
            pi += 1
    sl = torch.tensor(lens, dtype=torch.int32)
    out = torch.zeros(B, Hq, D)
    unified_attention(q.float(), kc, vc, out, torch.arange(B + 1, dtype=torch.int32), 1, sl, max(lens), D ** -0.5,
                      True, (-1, -1), bt, 0, None, torch.tensor([k_scale]), torch.tensor([v_scale]),
                      kv_quant_mode=KVQuantMode.FP8_PER_TENSOR)
    u8 = lambda x: x.view(torch.uint8).numpy()  # noqa: E731
    np.savez_compressed(OUT / f"{name}.npz", kind="decode_fp8", q=bits(q), k_cache=u8(kc), v_cache=u8(vc),
                        block_table=bt.numpy(), seq_lens=sl.numpy(), k_scale=np.float64(k_scale),
                        v_scale=np.float64(v_scale), out=out.numpy().astype(np.float32),
                        source="vllm-0.22.0 triton_unified_attention FP8_PER_TENSOR (TRITON_INTERPRET=1, fp32 q "
                        "storage of bf16 values)")
    print(name, "B", B, "out|max|", float(out.abs().max()))


def main():
    if "--fp8" in sys.argv:  # only the fp8 fixture (the others are committed)
        decode_fp8_case("decode_fp8_gqa4", [1, 33, 250, 16], Hq=32, Hkv=8, seed=6)
        return
    prefill_case("prefill_varlen_gqa4", [1, 7, 64, 130], Hq=8, Hkv=2, seed=1)
    prefill_case("prefill_single_200_gqa4", [200], Hq=4, Hkv=1, seed=2)
    prefill_case("prefill_mha", [33, 129], Hq=2, Hkv=2, seed=3)
    decode_case("decode_ragged_gqa4", [1, 17, 200, 64], Hq=8, Hkv=2, seed=4)
    decode_case("decode_gqa8_bs32", [300, 45], Hq=16, Hkv=2, bs=32, seed=5)
    decode_fp8_case("decode_fp8_gqa4", [1, 33, 250, 16], Hq=32, Hkv=8, seed=6)


if __name__ == "__main__":
    sys.exit(main())
