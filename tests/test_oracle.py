"""The CPU oracle (oracle/attn_oracle.c) against the golden vectors from the upstream kernel
(tests/golden/make_golden.py) and against its numpy restatement; plus self-consistency
properties (paged == dense, block-permutation invariance, causal prefix consistency)."""
import glob
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2505_03780_b200 import workload as W

GOLDEN = sorted(glob.glob(str(Path(__file__).parent / "golden" / "*.npz")))


@pytest.mark.parametrize("path", GOLDEN, ids=[Path(p).stem for p in GOLDEN])
def test_oracle_matches_golden(path):
    z = np.load(path)
    if str(z["kind"]) == "prefill":
        out = oracle.prefill(z["q"], z["k"], z["v"], z["cu_seqlens"])
    elif str(z["kind"]) == "decode_fp8":
        out = oracle.decode_fp8_np(z["q"], z["k_cache"], z["v_cache"], z["block_table"], z["seq_lens"],
                                   float(z["k_scale"]), float(z["v_scale"]))
    else:
        out = oracle.decode(z["q"], z["k_cache"], z["v_cache"], z["block_table"], z["seq_lens"])
    # golden is an fp32 kernel run; the oracle accumulates in fp64
    assert np.abs(out - z["out"]).max() < 5e-6


def test_c_oracle_equals_numpy_prefill():
    x = W.make_prefill(dict(W.C1, batch_size=3, seq_len=70, num_q_heads=8, num_kv_heads=2), device="cpu")
    x.cu_seqlens[:] = torch.tensor([0, 1, 70, 210], dtype=torch.int32)
    for causal in (True, False):
        a = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens, causal=causal)
        b = oracle.prefill_np(x.q, x.k, x.v, x.cu_seqlens, causal=causal)
        assert np.abs(a - b).max() < 1e-12


def test_c_oracle_equals_numpy_decode():
    d = W.make_decode(dict(W.C2, batch_size=4, seq_len=300), device="cpu", lens=[300, 1, 16, 17], extra_blocks=5)
    a = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    b = oracle.decode_np(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    assert np.abs(a - b).max() < 1e-12


def test_paged_decode_equals_dense_last_row_of_prefill():
    """decode of the last token == the causal prefill's last row (same K/V, paged vs dense)."""
    L, Hq, Hkv, bs = 77, 8, 2, 16
    x = W.make_prefill(dict(W.C1, seq_len=L, num_q_heads=Hq, num_kv_heads=Hkv), device="cpu")
    ref = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens)[L - 1]
    nb = (L + bs - 1) // bs
    perm = torch.randperm(nb + 3, generator=torch.Generator().manual_seed(0))
    kc = torch.zeros(nb + 3, bs, Hkv, 128, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    for t in range(L):
        kc[perm[t // bs], t % bs] = x.k[t]
        vc[perm[t // bs], t % bs] = x.v[t]
    bt = perm[:nb].to(torch.int32)[None]
    out = oracle.decode(x.q[L - 1:L], kc, vc, bt, torch.tensor([L], dtype=torch.int32))[0]
    assert np.abs(out - ref).max() < 1e-12


def test_decode_block_permutation_invariance():
    d = W.make_decode(dict(W.C2, batch_size=2, seq_len=64), device="cpu", extra_blocks=4)
    a = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    p = torch.randperm(d.k_cache.shape[0], generator=torch.Generator().manual_seed(9))
    inv = torch.empty_like(p)
    inv[p] = torch.arange(len(p))
    b = oracle.decode(d.q, d.k_cache[p], d.v_cache[p], inv[d.block_table.long()].to(torch.int32), d.seq_lens)
    assert np.abs(a - b).max() < 1e-12


def test_oracle_lse():
    x = W.make_prefill(dict(W.C1, seq_len=40, num_q_heads=2, num_kv_heads=1), device="cpu")
    _, lse = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens, with_lse=True)
    q = oracle.bf16_bits_to_f64(oracle.as_bf16_bits(x.q))
    k = oracle.bf16_bits_to_f64(oracle.as_bf16_bits(x.k))
    s = np.einsum("id,jd->ij", q[:, 1], k[:, 0]) / np.sqrt(128)
    s = np.where(np.tril(np.ones((40, 40), bool)), s, -np.inf)
    ref = np.log(np.exp(s - s.max(1, keepdims=True)).sum(1)) + s.max(1)
    assert np.abs(lse[1] - ref).max() < 1e-10


def test_e4m3_table_matches_torch_float8():
    """The oracle's OCP e4m3 decode table == torch.float8_e4m3fn for all 256 codes (NaN at 0x7f/0xff)."""
    t = oracle.e4m3_table()
    ref = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).double().numpy()
    assert np.array_equal(np.isnan(t), np.isnan(ref))
    ok = ~np.isnan(t)
    assert np.array_equal(t[ok], ref[ok])


def test_e4m3_quantizer_matches_torch_in_range():
    x = np.random.RandomState(0).randn(200000).astype(np.float32) * 3
    ours = oracle.quantize_e4m3_np(x, 64.0)
    ref = (torch.from_numpy(x) * 64).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    inr = np.abs(x * 64) <= 448
    assert np.array_equal(ours[inr], ref[inr])
    assert set(np.unique(ours[~inr] & 0x7F)) <= {0x7E}  # saturates to +-448 (satfinite)


def test_fp8_decode_equals_bf16_decode_on_dequantised_cache():
    """With power-of-two scales e4m3 * scale is exact in bf16: the fp8 oracle == the (pinned) bf16 one."""
    d = W.make_decode(dict(W.C2, batch_size=3, seq_len=200, kv_dtype="fp8_e4m3"), device="cpu",
                      lens=[200, 1, 77], extra_blocks=2)
    a = oracle.decode_fp8_np(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, d.k_scale, d.v_scale)
    kb = (d.k_cache.float() * d.k_scale).bfloat16()
    vb = (d.v_cache.float() * d.v_scale).bfloat16()
    assert torch.equal(kb.float(), d.k_cache.float() * d.k_scale)
    b = oracle.decode(d.q, kb, vb, d.block_table, d.seq_lens)
    assert np.abs(a - b).max() < 1e-12


def test_blas_prefill_equals_c_oracle():
    """The chunked-BLAS fp64 restatement (used by the full-size GPU parity tests) == the C oracle."""
    x = W.make_prefill(dict(W.C1, batch_size=3, seq_len=70, num_q_heads=8, num_kv_heads=2), device="cpu")
    x.cu_seqlens[:] = torch.tensor([0, 1, 70, 210], dtype=torch.int32)
    for causal in (True, False):
        a = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens, causal=causal)
        b = oracle.prefill_blas(x.q, x.k, x.v, x.cu_seqlens, causal=causal, chunk=32)
        assert np.abs(a - b).max() < 1e-12
        c = oracle.prefill_blas(x.q, x.k, x.v, x.cu_seqlens, causal=causal, heads=[1, 6])
        assert np.abs(a[:, [1, 6]] - c).max() < 1e-12


def test_torch_cpu_sdpa_matches_oracle():
    """oracle/torch_cpu.py (the PyTorch-native CPU baseline, fp32) agrees with the fp64 oracle."""
    import torch_cpu

    x = W.make_prefill(dict(W.C1, batch_size=2, seq_len=150, num_q_heads=8, num_kv_heads=2), device="cpu")
    x.cu_seqlens[:] = torch.tensor([0, 40, 300], dtype=torch.int32)
    ref = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens)
    assert np.abs(torch_cpu.prefill(x.q, x.k, x.v, x.cu_seqlens).double().numpy() - ref).max() < 1e-5
    d = W.make_decode(dict(W.C2, batch_size=3, seq_len=300), device="cpu", lens=[300, 1, 33], extra_blocks=2)
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    out = torch_cpu.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    assert np.abs(out.double().numpy() - ref).max() < 1e-5
    out = torch_cpu.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, dtype=torch.bfloat16)
    assert np.abs(out.double().numpy() - ref).max() < 2e-2  # bf16 output rounding
