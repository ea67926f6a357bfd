"""GPU parity: the sm_100a kernels (through the C ABI) vs the CPU oracle on identical inputs.

Tolerance (bf16 in, fp32 accumulate, bf16 out), per case:
  * max-abs error <= 2 x (max-abs error of torch SDPA run in bf16 on the same inputs) + 1e-4;
  * max-abs error <= 1e-2 beyond the bf16 output quantum: every element satisfies
    |out - ref| <= 1e-2 + ulp_bf16(ref) / 2.  The plain max-abs <= 1e-2 is asserted on every
    BASELINE configuration (C1, C2, C3, C4) and golden vector wherever torch SDPA in bf16 meets it
    on the same inputs; where SDPA-bf16 itself misses it (the full C3 has outputs with |O| > 2,
    where one bf16 ulp is >= 1.6e-2; SDPA's max-abs there is 1.03e-2, identical to ours), the
    quantum-aware form is asserted instead.  Synthetic edge cases that drive |O| past 2 use the
    quantum-aware form, and the adversarial score-jump inputs, on which SDPA-bf16 misses 1e-2 even
    beyond the quantum, are held to the 2x-SDPA bound alone — BASELINE.md §4 amendment;
  * max-rel error = max |out - ref| / max(|ref|, 1) <= 1e-2.
Errors are printed per case (pytest -s) and tabulated at the end of the run (tests/conftest.py).
Full-size configs are checked IN FULL against the oracle: C1, C2 (all 64 sequences), C3 (all 16
sequences x 32 q heads, through the BLAS fp64 restatement), a 32-sequence C4 shard (the per-GPU
load at 8 GPUs), and the whole 256-sequence C4 on one GPU on a seeded subset; plus properties:
split-count invariance, physical-page permutation invariance (bit-exact).
"""
import glob
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
from paper_2505_03780_b200 import attention as A
from paper_2505_03780_b200 import workload as W

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
DEV = "cuda"


def pcfg(bm=256, bn=128, ns=3, pre=False, nw=4, pair=False):
    """pair: waves_per_eu = 2, the work item on a CTA pair (cta_group::2, M = 256 MMAs)."""
    return dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=nw, num_stages=ns, waves_per_eu=2 if pair else 1, PRE_LOAD_V=pre)


def dcfg(splits=0, ns=4, tile=128):
    return dict(num_splits=splits, num_stages=ns, TILE_N=tile)


FLAT = dcfg(0, 4, 16)
DECODE_CFGS = [dcfg(1), dcfg(4), dcfg(0), dcfg(0, 4, 16), dcfg(0, 3, 16)]


def sdpa_prefill_bf16(q, k, v, cu, causal):
    outs = []
    G = q.shape[1] // k.shape[1]
    for s in range(len(cu) - 1):
        a, b = int(cu[s]), int(cu[s + 1])
        if b == a:
            continue
        qq = q[a:b].transpose(0, 1)[None]
        kk = k[a:b].repeat_interleave(G, 1).transpose(0, 1)[None]
        vv = v[a:b].repeat_interleave(G, 1).transpose(0, 1)[None]
        outs.append(F.scaled_dot_product_attention(qq, kk, vv, is_causal=causal)[0].transpose(0, 1))
    return torch.cat(outs).float().cpu().numpy()


def sdpa_decode_bf16(q, kc, vc, bt, sl):
    B, Hq, D = q.shape
    G = Hq // kc.shape[2]
    bs = kc.shape[1]
    out = torch.zeros(B, Hq, D)
    for b in range(B):
        n = int(sl[b])
        t = torch.arange(n, device=q.device)
        pages = bt[b, t // bs].long()
        kk = kc[pages, t % bs].repeat_interleave(G, 1).transpose(0, 1)[None]
        vv = vc[pages, t % bs].repeat_interleave(G, 1).transpose(0, 1)[None]
        out[b] = F.scaled_dot_product_attention(q[b][None, :, None], kk, vv)[0, :, 0].float().cpu()
    return out.numpy()


PARITY_TOL = 1e-2
RESULTS = []  # (name, max_abs, max_rel, sdpa_bf16_max_abs, max_abs_beyond_quantum, bound) -> conftest summary


def bf16_half_ulp(x: np.ndarray) -> np.ndarray:
    """half the spacing of bf16 numbers at |x| (8 significant bits)."""
    e = np.floor(np.log2(np.maximum(np.abs(x), 2.0 ** -126)))
    return 2.0 ** (e - 8)


def check(name, out, ref, base, strict=False):
    """strict (BASELINE configs, goldens): plain max-abs <= 1e-2 wherever SDPA-bf16 meets it.
    Otherwise the 1e-2 bound applies beyond bf16's own output rounding (see module docstring)."""
    out = out.float().cpu().numpy() if isinstance(out, torch.Tensor) else out
    err = np.abs(out - ref)
    base_err = np.abs(base - ref).max()
    rel = (err / np.maximum(np.abs(ref), 1.0)).max()
    beyond = (err - bf16_half_ulp(ref)).max()
    if strict and base_err <= PARITY_TOL:
        bound = "max_abs<=1e-2"
    elif strict or base_err <= PARITY_TOL:
        bound = "beyond-quantum<=1e-2"
    else:  # bf16 arithmetic itself (SDPA) misses 1e-2 beyond the quantum: the 2x-SDPA bound rules
        bound = "2x-sdpa only"
    print(f"[parity] {name}: max_abs={err.max():.3e} max_rel={rel:.3e} mean_abs={err.mean():.2e} "
          f"sdpa_bf16_max_abs={base_err:.3e} beyond_bf16_quantum={beyond:.3e} bound={bound}")
    RESULTS.append((name, float(err.max()), float(rel), float(base_err), float(beyond), bound))
    assert not np.isnan(out).any(), name
    assert err.max() <= 2 * base_err + 1e-4, (name, err.max(), base_err)
    assert rel <= 1e-2, (name, rel)
    if bound == "max_abs<=1e-2":
        assert err.max() <= PARITY_TOL, (name, err.max())
    elif bound == "beyond-quantum<=1e-2":
        assert beyond <= PARITY_TOL, (name, beyond)


def run_prefill(lens, Hq=32, Hkv=8, causal=True, cfg=None, seed=1):
    g = torch.Generator().manual_seed(seed)
    T = sum(lens)
    q = torch.randn(T, Hq, 128, generator=g).bfloat16()
    k = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    v = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref = oracle.prefill(q, k, v, cu, causal=causal)
    qd, kd, vd = q.to(DEV), k.to(DEV), v.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cu.to(DEV), max(lens), causal=causal, config=cfg)
    base = sdpa_prefill_bf16(qd, kd, vd, cu, causal)
    return out, ref, base


# ------------------------------------------------------------------ tcgen05 descriptor self-test
@pytest.mark.parametrize("mode", [0, 1, 2, 3])
def test_umma_selftest(mode):
    g = torch.Generator().manual_seed(mode)
    a = torch.randn(128, 128, generator=g).bfloat16().to(DEV)
    b = torch.randn(16 if mode == 2 else 128, 128, generator=g).bfloat16().to(DEV)
    d = A.selftest_umma(mode, a, b)
    af, bf = a.double(), b.double()
    ref = af @ bf.t() if mode in (0, 3) else (af @ bf if mode == 1 else af.t() @ bf.t())
    assert (d.double() - ref).abs().max().item() < 1e-3


@pytest.mark.parametrize("mode", [4, 5])
def test_umma_selftest_fp8(mode):
    """kind::f8f6f4 descriptors: e4m3 A (K-major, or MN-major given as [K][M]) x e4m3 B K-major."""
    g = torch.Generator().manual_seed(mode)
    a = (torch.randn(128, 128, generator=g) * 8).to(torch.float8_e4m3fn)
    b = (torch.randn(128, 128, generator=g) * 8).to(torch.float8_e4m3fn)
    d = A.selftest_umma(mode, a.view(torch.uint8).to(DEV), b.view(torch.uint8).to(DEV))
    af, bf = a.double(), b.double()
    ref = af @ bf.t() if mode == 4 else af.t() @ bf.t()
    assert (d.double().cpu() - ref).abs().max().item() < 1e-2 * ref.abs().max().item()


# ------------------------------------------------------------------ golden fixtures (upstream kernel)
GOLDEN = sorted(glob.glob(str(ROOT / "tests" / "golden" / "*.npz")))


def _t(bits, shape=None):
    return torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16)


@pytest.mark.parametrize("path", GOLDEN, ids=[Path(p).stem for p in GOLDEN])
def test_golden(path):
    z = np.load(path)
    if str(z["kind"]) == "prefill":
        q, k, v = (_t(z[n]).to(DEV) for n in ("q", "k", "v"))
        cu = torch.from_numpy(z["cu_seqlens"]).to(DEV)
        lens = np.diff(z["cu_seqlens"])
        cfg = pcfg() if (q.shape[1] // k.shape[1]) % 2 == 0 else pcfg(bm=128)
        out = A.prefill_varlen(q, k, v, cu, int(lens.max()), config=cfg)
        base = sdpa_prefill_bf16(q, k, v, z["cu_seqlens"], True)
    elif str(z["kind"]) == "decode_fp8":
        q = _t(z["q"]).to(DEV)
        kc, vc = (torch.from_numpy(z[n]).view(torch.float8_e4m3fn).to(DEV) for n in ("k_cache", "v_cache"))
        bt = torch.from_numpy(z["block_table"]).to(DEV)
        sl = torch.from_numpy(z["seq_lens"]).to(DEV)
        ks, vs = float(z["k_scale"]), float(z["v_scale"])
        out = A.paged_decode(q, kc, vc, bt, sl, k_scale=ks, v_scale=vs)
        base = sdpa_decode_bf16(q, (kc.float() * ks).bfloat16(), (vc.float() * vs).bfloat16(), bt, sl)
    else:
        q, kc, vc = (_t(z[n]).to(DEV) for n in ("q", "k_cache", "v_cache"))
        bt = torch.from_numpy(z["block_table"]).to(DEV)
        sl = torch.from_numpy(z["seq_lens"]).to(DEV)
        out = A.paged_decode(q, kc, vc, bt, sl)
        base = sdpa_decode_bf16(q, kc, vc, bt, sl)
    check(Path(path).stem, out, z["out"].astype(np.float64), base, strict=True)


# ------------------------------------------------------------------ prefill
@pytest.mark.parametrize("lens", [[512], [128], [1], [200], [1, 5, 127, 128, 129, 300], [64, 1000, 3]],
                         ids=lambda l: "x".join(map(str, l)))
def test_prefill_causal(lens):
    out, ref, base = run_prefill(lens)
    check(f"prefill {lens}", out, ref, base)


@pytest.mark.parametrize("nw", [4, 8])
@pytest.mark.parametrize("boost", [6.0, 40.0])
@pytest.mark.parametrize("start", [256, 320], ids=["jump_lo_half", "jump_hi_half"])
def test_prefill_score_jumps_after_first_tile(boost, nw, start):
    """Keys past `start` are scaled up so later tiles' scores exceed the running max from the first
    tile by ~20 (boost 6: the speculative single pass keeps P = 2^(s - m_run) up to 2^20 in bf16) or
    by > 64 (boost 40: the row sum passes 2^64 and the tile is redone exactly); start = 320 puts
    the jump in the upper half of a 128-key tile."""
    g = torch.Generator().manual_seed(7)
    lens = [1000, 640]
    T, Hq, Hkv = sum(lens), 16, 4
    q = torch.randn(T, Hq, 128, generator=g).bfloat16()
    k = torch.randn(T, Hkv, 128, generator=g)
    k[start:1000] *= boost
    k[1000 + start:] *= boost
    k = k.bfloat16()
    v = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref = oracle.prefill(q, k, v, cu)
    qd, kd, vd = q.to(DEV), k.to(DEV), v.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cu.to(DEV), max(lens), config=pcfg(ns=2 if nw == 8 else 3, nw=nw))
    assert not torch.isnan(out).any()
    check(f"prefill score jumps x{boost} w{nw} from {start}", out, ref, sdpa_prefill_bf16(qd, kd, vd, cu, True))


@pytest.mark.parametrize("boost", [6.0, 40.0])
@pytest.mark.parametrize("start", [256, 320], ids=["jump_lo_half", "jump_hi_half"])
def test_prefill_score_jumps_block_m_128(boost, start):
    """The same with one q head per CTA (BLOCK_M = 128: S double-buffered, QK two KV steps ahead)."""
    g = torch.Generator().manual_seed(8)
    lens = [900, 500]
    T, Hq, Hkv = sum(lens), 8, 2
    q = torch.randn(T, Hq, 128, generator=g).bfloat16()
    k = torch.randn(T, Hkv, 128, generator=g)
    k[start:900] *= boost
    k[900 + start:] *= boost
    k = k.bfloat16()
    v = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref = oracle.prefill(q, k, v, cu)
    qd, kd, vd = q.to(DEV), k.to(DEV), v.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cu.to(DEV), max(lens), config=pcfg(bm=128, ns=3))
    assert not torch.isnan(out).any()
    check(f"prefill score jumps bm128 x{boost} from {start}", out, ref, sdpa_prefill_bf16(qd, kd, vd, cu, True))


@pytest.mark.parametrize("nw", [4, 8])
def test_prefill_noncausal(nw):
    out, ref, base = run_prefill([200, 64, 129], causal=False, cfg=pcfg(ns=2, nw=nw))
    check(f"prefill noncausal w{nw}", out, ref, base)


@pytest.mark.parametrize("nw", [4, 8])
@pytest.mark.parametrize("hq,hkv", [(8, 8), (16, 2), (32, 8), (64, 8)])
def test_prefill_gqa_shapes(hq, hkv, nw):
    cfg = pcfg(bm=128, ns=2, nw=nw) if (hq // hkv) % 2 else pcfg(ns=2, nw=nw)
    out, ref, base = run_prefill([300, 17], Hq=hq, Hkv=hkv, cfg=cfg)
    check(f"prefill gqa {hq}/{hkv} w{nw}", out, ref, base)


VARIANTS = [(bm, bn, ns, 4, False) for bm in (128, 256) for bn in (64, 128) for ns in (1, 2, 3, 4)] + \
    [(bm, 128, ns, 8, False) for bm in (128, 256) for ns in (1, 2)] + \
    [(bm, 128, ns, 4, True) for bm in (128, 256) for ns in (1, 2, 3)]


@pytest.mark.parametrize("bm,bn,ns,nw,pair", VARIANTS)
def test_prefill_every_compiled_variant(bm, bn, ns, nw, pair):
    out, ref, base = run_prefill([300, 77, 129], cfg=pcfg(bm, bn, ns, nw=nw, pair=pair))
    check(f"prefill variant {bm}/{bn}/{ns}/w{nw}{'/pair' if pair else ''}", out, ref, base)


@pytest.mark.parametrize("cfg", [pcfg(), pcfg(128, 128, 3), pcfg(256, 128, 2, nw=8), pcfg(256, 128, 2, pair=True)],
                         ids=["bm256", "bm128", "bm256w8", "pair"])
@pytest.mark.parametrize("lens", [[128] * 16, [300] * 5, [1] * 7, [1024] * 3], ids=lambda l: f"{len(l)}x{l[0]}")
def test_prefill_uniform_batch(cfg, lens):
    """Equal-length batches take the analytic item order (no schedule kernel): ragged last q blocks,
    single tokens, many short sequences; causal and not."""
    for causal in (True, False):
        out, ref, base = run_prefill(lens, cfg=cfg, causal=causal)
        check(f"prefill uniform {len(lens)}x{lens[0]} causal={causal}", out, ref, base)


# ------------------------------------------------------------------ CTA pair (cta_group::2) variants
PAIR_CFGS = [pcfg(256, 128, 2, pair=True), pcfg(128, 128, 2, pair=True)]


@pytest.mark.parametrize("cfg", PAIR_CFGS, ids=["pair_bm256", "pair_bm128"])
@pytest.mark.parametrize("lens", [[1], [128], [129], [512], [1, 5, 127, 128, 129, 300], [2000, 64, 3]],
                         ids=lambda l: "x".join(map(str, l)) if isinstance(l, list) else None)
def test_prefill_pair_ragged(cfg, lens):
    """The pair splits every K tile by keys (64 per CTA) and every V tile by d columns: ragged tails,
    single tokens and sequences shorter than one CTA's K half."""
    out, ref, base = run_prefill(lens, cfg=cfg)
    check(f"prefill pair bm{cfg['BLOCK_M']} {lens}", out, ref, base)


@pytest.mark.parametrize("cfg", PAIR_CFGS, ids=["pair_bm256", "pair_bm128"])
@pytest.mark.parametrize("hq,hkv", [(16, 2), (32, 8), (64, 8), (8, 2)])
def test_prefill_pair_gqa_and_noncausal(cfg, hq, hkv):
    if (hq // hkv) % (2 * cfg["BLOCK_M"] // 128):
        pytest.skip("group not a multiple of the pair's q heads (reported as invalid)")
    for causal in (True, False):
        out, ref, base = run_prefill([300, 17, 256], Hq=hq, Hkv=hkv, causal=causal, cfg=cfg)
        check(f"prefill pair bm{cfg['BLOCK_M']} gqa {hq}/{hkv} causal={causal}", out, ref, base)


@pytest.mark.parametrize("boost", [6.0, 40.0])
def test_prefill_pair_score_jumps(boost):
    g = torch.Generator().manual_seed(9)
    lens = [1000, 640]
    T, Hq, Hkv = sum(lens), 16, 4
    q = torch.randn(T, Hq, 128, generator=g).bfloat16()
    k = torch.randn(T, Hkv, 128, generator=g)
    k[320:1000] *= boost
    k[1000 + 256:] *= boost
    k = k.bfloat16()
    v = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref = oracle.prefill(q, k, v, cu)
    qd, kd, vd = q.to(DEV), k.to(DEV), v.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cu.to(DEV), max(lens), config=PAIR_CFGS[0])
    assert not torch.isnan(out).any()
    check(f"prefill pair score jumps x{boost}", out, ref, sdpa_prefill_bf16(qd, kd, vd, cu, True))


def test_prefill_pair_lse_and_repeat():
    """LSE from both CTAs of the pair, and bit-identical results over repeated launches (the pair's
    barriers and the self-resetting work counter carry no state between launches)."""
    lens = [100, 257, 1100]
    g = torch.Generator().manual_seed(4)
    T = sum(lens)
    q, k, v = (torch.randn(T, h, 128, generator=g).bfloat16() for h in (16, 4, 4))
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref, ref_lse = oracle.prefill(q, k, v, cu, with_lse=True)
    args = (q.to(DEV), k.to(DEV), v.to(DEV), cu.to(DEV), max(lens))
    out, lse = A.prefill_varlen(*args, return_lse=True, config=PAIR_CFGS[0])
    assert np.abs(lse.cpu().numpy() - ref_lse).max() < 2e-3
    assert np.abs(out.float().cpu().numpy() - ref).max() < 2e-2
    for _ in range(3):
        assert torch.equal(A.prefill_varlen(*args, config=PAIR_CFGS[0]), out)


@pytest.mark.parametrize("cfg", [None, pcfg(256, 128, 2, nw=8), pcfg(128, 128, 1, nw=8)], ids=["default", "bm256w8", "bm128w8"])
def test_prefill_lse(cfg):
    lens = [100, 257]
    g = torch.Generator().manual_seed(3)
    T = sum(lens)
    q, k, v = (torch.randn(T, h, 128, generator=g).bfloat16() for h in (8, 2, 2))
    cu = torch.tensor([0, 100, 357], dtype=torch.int32)
    ref, ref_lse = oracle.prefill(q, k, v, cu, with_lse=True)
    out, lse = A.prefill_varlen(q.to(DEV), k.to(DEV), v.to(DEV), cu.to(DEV), 257, return_lse=True, config=cfg)
    assert np.abs(lse.cpu().numpy() - ref_lse).max() < 2e-3
    assert np.abs(out.float().cpu().numpy() - ref).max() < 2e-2


def test_prefill_c1_full():
    x = W.make_prefill(W.C1, device="cpu")
    ref = oracle.prefill(x.q, x.k, x.v, x.cu_seqlens)
    qd, kd, vd = x.q.to(DEV), x.k.to(DEV), x.v.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, x.cu_seqlens.to(DEV), x.max_seqlen)
    check("C1 full", out, ref, sdpa_prefill_bf16(qd, kd, vd, x.cu_seqlens, True), strict=True)


@pytest.mark.parametrize("cfg", [None, pcfg(256, 128, 2, nw=8), pcfg(256, 128, 2, pair=True)],
                         ids=["dispatch", "bm256w8", "pair"])
def test_prefill_c3_full(cfg):
    """All of C3 (16 seqs, 33430 tokens, 32 q heads) on the GPU vs the fp64 oracle on EVERY
    sequence and head (oracle.prefill_blas: the BLAS restatement, pinned to the C oracle in
    tests/test_oracle.py).  SDPA-bf16's error is computed on the same full problem."""
    x = W.make_prefill(W.C3, device="cpu")
    qd, kd, vd, cud = x.q.to(DEV), x.k.to(DEV), x.v.to(DEV), x.cu_seqlens.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cud, x.max_seqlen, config=cfg).cpu()
    ref = oracle.prefill_blas(x.q, x.k, x.v, x.cu_seqlens)
    base = sdpa_prefill_bf16(qd, kd, vd, x.cu_seqlens, True)
    tag = "dispatch" if cfg is None else ("pair" if cfg["waves_per_eu"] == 2 else "bm256w8")
    check(f"C3 full (16 seqs x 32 heads) {tag}", out, ref, base, strict=True)


# ------------------------------------------------------------------ decode
def run_decode(lens, Hq=32, Hkv=8, bs=16, cfg=None, seed=0):
    shape = dict(W.C2, batch_size=len(lens), seq_len=max(lens), num_q_heads=Hq, num_kv_heads=Hkv, block_size=bs,
                 seed=seed)
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=3)
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=cfg)
    return out, ref, sdpa_decode_bf16(*args)


@pytest.mark.parametrize("lens", [[1], [128], [4096, 4096], [1, 15, 16, 17, 127, 128, 129, 1000]],
                         ids=lambda l: "x".join(map(str, l)))
@pytest.mark.parametrize("cfg", DECODE_CFGS, ids=lambda c: f"tile{c['TILE_N']}_s{c['num_splits']}_ns{c['num_stages']}")
def test_decode_ragged(lens, cfg):
    out, ref, base = run_decode(lens, cfg=cfg)
    check(f"decode {lens} {cfg}", out, ref, base)


@pytest.mark.parametrize("lens,hq", [
    ([8000], 32),                        # 1 x 32 = 32 merge CTAs -> (8 warps, 8 pieces in flight); ~128 pieces
    ([3000, 1, 700, 2048, 16, 5000], 32),  # 192 merge CTAs -> (8, 4), ragged, a 1-token sequence
    ([500, 37, 1500, 800] * 10, 16),     # 40 x 16 = 640 merge CTAs -> (4, 1)
    ([20000, 3], 8),                     # GQA 8/8 (G = 1): 16 merge CTAs, a sequence over every CTA
], ids=["1x8000", "6ragged", "40x_hq16", "hq8_long"])
def test_decode_flat_single_pass_merge_shapes(lens, hq):
    """K3' (single-pass online merge) in each of its three launch shapes — (warps, pieces in flight)
    = (8, 8) / (8, 4) / (4, 1) picked by the grid size — against the oracle, and bit-identical on a
    second launch (fixed fold order)."""
    cfg = dcfg(0, 4, 16)
    out, ref, base = run_decode(lens, Hq=hq, cfg=cfg)
    check(f"decode flat K3' shape {len(lens)}x{max(lens)} hq={hq}", out, ref, base)
    out2, _, _ = run_decode(lens, Hq=hq, cfg=cfg)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("splits", [2, 7, 16])
def test_decode_split_single_pass_merge(splits):
    """K3 (split-KV path, single-pass merge over 8 splits per round) at 2 / 7 / 16 splits vs the oracle."""
    out, ref, base = run_decode([3000, 1, 900, 129], cfg=dcfg(splits, 4, 128))
    check(f"decode K2 splits={splits}", out, ref, base)


@pytest.mark.parametrize("bs", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("tile", [16, 128])
def test_decode_block_sizes(bs, tile):
    if tile == 16 and bs < 16:
        pytest.skip("TILE_N=16 needs block_size >= 16 (reported as invalid)")
    out, ref, base = run_decode([700, 3000, 5], bs=bs, cfg=dcfg(0, 4, tile))
    check(f"decode bs={bs} tile={tile}", out, ref, base)


@pytest.mark.parametrize("hq,hkv", [(8, 8), (16, 8), (32, 8), (64, 8), (16, 1)])
def test_decode_gqa(hq, hkv):
    out, ref, base = run_decode([700, 130], Hq=hq, Hkv=hkv)  # default config (flat where compiled)
    check(f"decode gqa {hq}/{hkv}", out, ref, base)


@pytest.mark.parametrize("ns", [2, 3, 4, 5, 6])
def test_decode_every_stage_count(ns):
    out, ref, base = run_decode([1000, 333], cfg=dcfg(2, ns))
    check(f"decode split stages={ns}", out, ref, base)


@pytest.mark.parametrize("hq,ns", [(8, 3), (8, 6), (16, 5), (32, 3), (32, 5), (64, 3), (64, 4)])
def test_decode_flat_every_variant(hq, ns):
    out, ref, base = run_decode([1000, 333, 17], Hq=hq, cfg=dcfg(0, ns, 16))
    check(f"decode flat hq={hq} stages={ns}", out, ref, base)


# K2' at Hkv < 8: PPT = 8 / Hkv page chunks per 128-row tile (the kv-head shards of GQA models)
NARROW = [(4, 4, 4), (4, 8, 4), (4, 16, 4), (4, 32, 4), (4, 8, 5), (4, 16, 5), (2, 2, 4), (2, 4, 4), (2, 8, 4),
          (2, 16, 4), (2, 8, 5), (2, 16, 5), (1, 1, 4), (1, 2, 4), (1, 4, 4), (1, 8, 4), (1, 8, 5)]


@pytest.mark.parametrize("hkv,hq,ns", NARROW, ids=lambda v: str(v))
def test_decode_flat_narrow_kv_heads(hkv, hq, ns):
    """every compiled Hkv = 1/2/4 flat variant; lengths that end mid-chunk, mid-tile and at 1."""
    out, ref, base = run_decode([1000, 333, 17, 1, 129], Hq=hq, Hkv=hkv, cfg=dcfg(0, ns, 16))
    check(f"decode flat hkv={hkv} hq={hq} stages={ns}", out, ref, base)


@pytest.mark.parametrize("hkv", [1, 2, 4])
@pytest.mark.parametrize("bs", [16, 32, 128])
def test_decode_flat_narrow_block_sizes_and_nan_tails(hkv, bs):
    """Hkv < 8 with pages of 16..128 tokens; slots past each sequence's end hold NaN (a tile's
    chunks past the end reload a live chunk and are masked; the V rows are zeroed before PV)."""
    lens = [33, 250, 16, 700]
    shape = dict(W.C2, batch_size=4, seq_len=700, num_q_heads=8 * hkv, num_kv_heads=hkv, block_size=bs)
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=2)
    kc, vc = d.k_cache.clone(), d.v_cache.clone()
    live = torch.zeros(kc.shape[0], bs, dtype=torch.bool)
    for b, n in enumerate(lens):
        for t in range(n):
            live[d.block_table[b, t // bs], t % bs] = True
    kc[~live] = float("nan")
    vc[~live] = float("nan")
    ref = oracle.decode(d.q, kc, vc, d.block_table, d.seq_lens)
    args = [t.to(DEV) for t in (d.q, kc, vc, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=dcfg(0, 4, 16))
    assert not torch.isnan(out).any()
    check(f"decode flat hkv={hkv} bs={bs} NaN tails", out, ref, sdpa_decode_bf16(*args))


def test_decode_flat_kv_head_shard_of_c4():
    """The C4 geometry sharded by kv head over 8 GPUs: each GPU holds Hkv = 1 with its 8 q heads
    (64q/8kv -> 8q/1kv), ctx 32k — K2' at PPT = 8, every sequence vs the oracle."""
    shape = dict(W.C4, batch_size=6, num_q_heads=8, num_kv_heads=1)
    d = W.make_decode(shape, device="cpu", lens=[32768, 32768, 32767, 20000, 4096, 1])
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    plan = A.DecodePlan(*args)
    assert plan.config["TILE_N"] == 16, plan.config  # the dispatcher picks the flat kernel for Hkv = 1
    out = plan.run()
    check("decode C4 kv-head shard (8q/1kv, 32k)", out, ref, sdpa_decode_bf16(*args))


def test_decode_flat_batch_above_1024():
    """3000 ragged sequences (batch > the 1024 fused-merge counters): the per-sequence tile prefix
    is sized per launch and split sequences are merged by K3'."""
    g = torch.Generator().manual_seed(5)
    lens = torch.randint(1, 400, (3000,), generator=g).tolist()
    lens[10] = 0
    lens[2999] = 5000
    shape = dict(W.C2, batch_size=len(lens), seq_len=max(lens))
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=1)
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=FLAT)
    assert out[10].abs().max().item() == 0
    sub = [0, 1, 500, 1023, 1024, 1025, 2000, 2998, 2999]
    ref = oracle.decode(d.q[sub], d.k_cache, d.v_cache, d.block_table[sub], d.seq_lens[sub])
    ki = torch.tensor(sub, device=DEV)
    base = sdpa_decode_bf16(args[0][ki], args[1], args[2], args[3][ki], args[4][ki])
    check("decode flat B=3000 ragged", out[sub], ref, base)


def test_decode_flat_many_short_sequences():
    """300 ragged sequences: every CTA range spans many sequences and pieces of sequences."""
    g = torch.Generator().manual_seed(11)
    lens = torch.randint(1, 600, (300,), generator=g).tolist()
    lens[5] = 0  # an empty sequence -> zeros
    lens[7] = 4000
    shape = dict(W.C2, batch_size=len(lens), seq_len=max(lens))
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=3)
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=FLAT)
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    assert out[5].abs().max().item() == 0
    keep = [i for i in range(len(lens)) if lens[i] > 0]
    ki = torch.tensor(keep, device=DEV)
    base = sdpa_decode_bf16(args[0][ki], args[1], args[2], args[3][ki], args[4][ki])
    check("decode flat 300 ragged seqs", out[keep], ref[keep], base)


def test_decode_flat_repeatable_and_workspace_shared_with_split():
    """B = 64 ragged (sequences split across 2-3 CTAs): repeated plan runs and interleaved
    split-kernel calls sharing the cached workspace give bit-identical output."""
    g = torch.Generator().manual_seed(21)
    lens = torch.randint(1, 3000, (64,), generator=g).tolist()
    lens[3] = 0
    d = W.make_decode(dict(W.C2, batch_size=64, seq_len=max(lens)), device="cuda", lens=lens, extra_blocks=4)
    plan = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=FLAT)
    first = plan.run().clone()
    for _ in range(3):
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=dcfg(4))  # split kernel
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=FLAT)
        assert torch.equal(plan.run(), first)
    assert first[3].abs().max().item() == 0
    sub = [0, 1, 2, 40, 63]
    ref = oracle.decode(d.q[sub].cpu(), d.k_cache.cpu(), d.v_cache.cpu(), d.block_table[sub].cpu(),
                        d.seq_lens[sub].cpu())
    check("decode flat B=64 ragged", first[sub], ref,
          sdpa_decode_bf16(d.q[sub], d.k_cache, d.v_cache, d.block_table[sub], d.seq_lens[sub]))


@pytest.mark.parametrize("tile", [16, 128])
def test_decode_nan_in_unused_page_slots(tile):
    """Cache slots past each sequence's end hold NaN: the output must not see them."""
    lens = [33, 250, 16]
    d = W.make_decode(dict(W.C2, batch_size=3, seq_len=250), device="cpu", lens=lens, extra_blocks=2)
    kc, vc = d.k_cache.clone(), d.v_cache.clone()
    bs = kc.shape[1]
    live = torch.zeros(kc.shape[0], bs, dtype=torch.bool)
    for b, n in enumerate(lens):
        for t in range(n):
            live[d.block_table[b, t // bs], t % bs] = True
    kc[~live] = float("nan")
    vc[~live] = float("nan")
    ref = oracle.decode(d.q, kc, vc, d.block_table, d.seq_lens)
    args = [t.to(DEV) for t in (d.q, kc, vc, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=dcfg(0, 4, tile))
    assert not torch.isnan(out).any()
    check(f"decode NaN tails tile={tile}", out, ref, sdpa_decode_bf16(*args))


def test_decode_c2_full_size():
    """C2 in full on the GPU, ALL 64 sequences vs the oracle (flat K2'+K3' and the split K2+K3
    paths); split-count invariance on all 64."""
    d = W.make_decode(W.C2, device="cpu")
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    outs = {s: A.paged_decode(*args, config=dcfg(s)).float() for s in (1, 2, 8, 0)}
    outs["flat"] = A.paged_decode(*args, config=FLAT).float()
    for s in (2, 8, 0, "flat"):
        assert (outs[s] - outs[1]).abs().max().item() < 2e-2
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    base = sdpa_decode_bf16(*args)
    check("C2 full (64 seqs) split", outs[0], ref, base, strict=True)
    check("C2 full (64 seqs) flat", outs["flat"], ref, base, strict=True)


def test_decode_c4_shard_full():
    """The per-GPU load of C4 at 8 GPUs — 32 sequences x ctx 32768, 64q/8kv (4.3 GB of K+V; each
    sequence spans ~5 of the flat partition's CTAs) — every sequence vs the oracle."""
    shape = dict(W.C4, batch_size=32)
    d = W.make_decode(shape, device=DEV)
    out = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    cpu = [t.cpu() for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    ref = oracle.decode(*cpu)
    sub = list(range(0, 32, 8))  # SDPA-bf16 reference error on a subset (it gathers per sequence)
    base = sdpa_decode_bf16(d.q[sub], d.k_cache, d.v_cache, d.block_table[sub], d.seq_lens[sub])
    err = np.abs(out.float().cpu().numpy() - ref)
    base_err = np.abs(base - ref[sub]).max()
    rel = (err / np.maximum(np.abs(ref), 1.0)).max()
    print(f"[parity] C4 shard (32 x 32k) all seqs: max_abs={err.max():.3e} max_rel={rel:.3e} "
          f"sdpa_bf16_max_abs(4 seqs)={base_err:.3e}")
    RESULTS.append(("C4 shard (32 x 32k, 64q/8kv) all 32 seqs", float(err.max()), float(rel), float(base_err),
                    float((err - bf16_half_ulp(ref)).max()), "max_abs<=1e-2"))
    assert err.max() <= PARITY_TOL and err.max() <= 2 * base_err + 1e-4 and rel <= 1e-2


def test_decode_c4_full_one_gpu_seeded_subset():
    """The whole C4 (256 sequences x 32k, 34.4 GB of K+V) on one B200 through the sharded builder
    (every sequence's content is a function of its global index); 8 sequences spread over the batch
    are rebuilt on the host from their seeds and checked against the oracle."""
    shape = dict(W.C4)
    d = W.make_decode_shard(shape, 0, 256, device=DEV)
    out = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens).cpu()
    del d
    torch.cuda.empty_cache()
    worst = 0.0
    for b in (0, 37, 100, 127, 128, 200, 254, 255):
        q, k, v = (t.cpu() for t in W.decode_sequence(shape, b, device=DEV))  # same generator as the shard
        nb = k.shape[0] // 16
        ref = oracle.decode(q[None], k.view(nb, 16, 8, 128), v.view(nb, 16, 8, 128),
                            torch.arange(nb, dtype=torch.int32)[None], torch.tensor([k.shape[0]], dtype=torch.int32))
        worst = max(worst, float(np.abs(out[b:b + 1].float().numpy() - ref).max()))
    print(f"[parity] C4 full (256 x 32k) 8 seeded seqs: max_abs={worst:.3e}")
    RESULTS.append(("C4 full (256 x 32k) 8 seeded seqs", worst, worst, float("nan"), worst, "max_abs<=1e-2"))
    assert worst <= PARITY_TOL


@pytest.mark.parametrize("tile", [16, 128])
def test_decode_page_permutation_is_bit_exact(tile):
    d = W.make_decode(dict(W.C2, batch_size=8, seq_len=1000), device="cuda", extra_blocks=16)
    cfg = dcfg(0, 4, tile)
    a = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=cfg)
    p = torch.randperm(d.k_cache.shape[0], generator=torch.Generator().manual_seed(1)).to(DEV)
    inv = torch.empty_like(p)
    inv[p] = torch.arange(len(p), device=DEV)
    b = A.paged_decode(d.q, d.k_cache[p].contiguous(), d.v_cache[p].contiguous(),
                       inv[d.block_table.long()].to(torch.int32), d.seq_lens, config=cfg)
    assert torch.equal(a, b)


def test_combine_kernel():
    rows, S = 37, 5
    g = torch.Generator().manual_seed(0)
    po = torch.randn(rows, S, 128, generator=g)
    m = torch.randn(rows, S, generator=g) * 4
    m[0, 1:] = -float("inf")
    l = torch.rand(rows, S, generator=g) + 0.5
    l[0, 1:] = 0
    ml = torch.stack([m, l], -1)
    out = torch.empty(rows, 128, dtype=torch.bfloat16, device=DEV)
    A.combine(po.to(DEV), ml.contiguous().to(DEV), out)
    w = torch.exp2(m - m.max(1, keepdim=True).values)
    ref = (w[..., None] * po).sum(1) / (w * l).sum(1, keepdim=True)
    assert (out.float().cpu() - ref).abs().max().item() < 2e-2


def test_cache_append_bit_exact():
    NB, bs, Hkv, N = 40, 16, 8, 50
    g = torch.Generator().manual_seed(0)
    kc = torch.randn(NB, bs, Hkv, 128, generator=g).bfloat16().to(DEV)
    vc = torch.randn(NB, bs, Hkv, 128, generator=g).bfloat16().to(DEV)
    nk = torch.randn(N, Hkv, 128, generator=g).bfloat16().to(DEV)
    nv = torch.randn(N, Hkv, 128, generator=g).bfloat16().to(DEV)
    slots = torch.randperm(NB * bs, generator=g)[:N].to(DEV)
    slots[3] = -1
    rk, rv = kc.clone().view(-1, Hkv, 128), vc.clone().view(-1, Hkv, 128)
    keep = slots >= 0
    rk[slots[keep]] = nk[keep]
    rv[slots[keep]] = nv[keep]
    A.cache_append(nk, nv, kc, vc, slots)
    assert torch.equal(kc.view(-1, Hkv, 128), rk) and torch.equal(vc.view(-1, Hkv, 128), rv)


def test_append_then_decode_equals_oracle():
    """Serving step: append the new token's K/V into its page, then decode (the §8(f) row 2 path)."""
    lens = [33, 300]
    d = W.make_decode(dict(W.C2, batch_size=2, seq_len=300), device="cpu", lens=lens, extra_blocks=2)
    kc, vc = d.k_cache.clone(), d.v_cache.clone()
    g = torch.Generator().manual_seed(5)
    nk, nv = (torch.randn(2, 8, 128, generator=g).bfloat16() for _ in range(2))
    bs = 16
    slots = torch.tensor([int(d.block_table[b, (lens[b] - 1) // bs]) * bs + (lens[b] - 1) % bs for b in range(2)])
    kc.view(-1, 8, 128)[slots] = nk
    vc.view(-1, 8, 128)[slots] = nv
    ref = oracle.decode(d.q, kc, vc, d.block_table, d.seq_lens)
    kd, vd = d.k_cache.to(DEV), d.v_cache.to(DEV)
    A.cache_append(nk.to(DEV), nv.to(DEV), kd, vd, slots.to(DEV))
    out = A.paged_decode(d.q.to(DEV), kd, vd, d.block_table.to(DEV), d.seq_lens.to(DEV))
    base = sdpa_decode_bf16(d.q.to(DEV), kd, vd, d.block_table.to(DEV), d.seq_lens.to(DEV))
    check("append+decode", out, ref, base)


# ------------------------------------------------------------------ fp8 (e4m3) KV cache
def run_decode_fp8(lens, Hq=32, cfg=None, seed=0, nan_tails=False, Hkv=8):
    shape = dict(W.C2, batch_size=len(lens), seq_len=max(lens), num_q_heads=Hq, num_kv_heads=Hkv, seed=seed,
                 kv_dtype="fp8_e4m3")
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=3)
    kc, vc = d.k_cache.clone(), d.v_cache.clone()
    if nan_tails:  # e4m3 NaN codes (0x7f / 0xff) in every slot no sequence owns
        bs = kc.shape[1]
        live = torch.zeros(kc.shape[0], bs, dtype=torch.bool)
        for b, n in enumerate(lens):
            for t in range(n):
                live[d.block_table[b, t // bs], t % bs] = True
        kc.view(torch.uint8)[~live] = 0x7F
        vc.view(torch.uint8)[~live] = 0xFF
    ref = oracle.decode_fp8_np(d.q, kc, vc, d.block_table, d.seq_lens, d.k_scale, d.v_scale)
    args = [t.to(DEV) for t in (d.q, kc, vc, d.block_table, d.seq_lens)]
    out = A.paged_decode(*args, config=cfg, k_scale=d.k_scale, v_scale=d.v_scale)
    kb = (args[1].float() * d.k_scale).bfloat16()
    vb = (args[2].float() * d.v_scale).bfloat16()
    if nan_tails:
        kb, vb = torch.nan_to_num(kb), torch.nan_to_num(vb)
    return out, ref, sdpa_decode_bf16(args[0], kb, vb, args[3], args[4])


@pytest.mark.parametrize("hq,ns", [(8, 4), (8, 6), (8, 8), (16, 4), (16, 6), (16, 8), (32, 4), (32, 6), (32, 8), (64, 4), (64, 6)])
def test_decode_fp8_every_variant(hq, ns):
    out, ref, base = run_decode_fp8([1000, 333, 17, 1], Hq=hq, cfg=dcfg(0, ns, 16))
    check(f"decode fp8 hq={hq} stages={ns}", out, ref, base)


@pytest.mark.parametrize("hkv,hq,ns", [(4, 8, 8), (4, 16, 8), (4, 32, 6), (2, 8, 8), (2, 16, 6), (1, 8, 8)],
                         ids=lambda v: str(v))
def test_decode_fp8_narrow_kv_heads(hkv, hq, ns):
    """fp8 K2' at Hkv < 8 (16-token chunks of Hkv heads per TMA box, PPT chunks per tile), NaN tails."""
    out, ref, base = run_decode_fp8([1000, 333, 17, 1], Hq=hq, Hkv=hkv, cfg=dcfg(0, ns, 16), nan_tails=True)
    assert not torch.isnan(out).any()
    check(f"decode fp8 hkv={hkv} hq={hq} stages={ns}", out, ref, base)


def test_decode_fp8_many_ragged_sequences_and_nan_tails():
    g = torch.Generator().manual_seed(3)
    lens = torch.randint(1, 700, (200,), generator=g).tolist()
    lens[9] = 3000
    out, ref, base = run_decode_fp8(lens, nan_tails=True)
    assert not torch.isnan(out).any()
    check("decode fp8 200 ragged seqs, NaN tails", out, ref, base)


def test_decode_fp8_c2_full_size_subset():
    d = W.make_decode(dict(W.C2, kv_dtype="fp8_e4m3"), device="cuda")
    out = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
    sub = [0, 31, 63]
    kc, vc = d.k_cache.cpu(), d.v_cache.cpu()
    ref = oracle.decode_fp8_np(d.q[sub].cpu(), kc, vc, d.block_table[sub].cpu(), d.seq_lens[sub].cpu(),
                               d.k_scale, d.v_scale)
    base = sdpa_decode_bf16(d.q[sub], (d.k_cache.float() * d.k_scale).bfloat16(),
                            (d.v_cache.float() * d.v_scale).bfloat16(), d.block_table[sub], d.seq_lens[sub])
    check("C2 fp8 full (3 seqs checked)", out[sub], ref, base)


def test_decode_fp8_split_config_is_invalid():
    d = W.make_decode(dict(W.C2, batch_size=2, seq_len=64, kv_dtype="fp8_e4m3"), device="cuda")
    with pytest.raises(A._native.B200AttnError) as e:
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=dcfg(0, 4, 128))
    assert e.value.invalid


def test_cache_append_fp8_bit_exact():
    NB, bs, Hkv, N = 40, 16, 8, 50
    g = torch.Generator().manual_seed(0)
    kc = torch.zeros(NB, bs, Hkv, 128, dtype=torch.float8_e4m3fn, device=DEV)
    vc = torch.zeros_like(kc)
    nk = (torch.randn(N, Hkv, 128, generator=g) * 2).bfloat16()
    nv = (torch.randn(N, Hkv, 128, generator=g) * 9).bfloat16()
    nk[0, 0, :4] = torch.tensor([1e6, -1e6, 0.0, -0.0])  # saturation and signed zero
    slots = torch.randperm(NB * bs, generator=g)[:N]
    slots[3] = -1
    ks, vs = 1 / 64, 0.05
    A.cache_append(nk.to(DEV), nv.to(DEV), kc, vc, slots.to(DEV), k_scale=ks, v_scale=vs)
    keep = slots >= 0
    ek = oracle.quantize_e4m3_np(nk.float().numpy() * np.float32(1 / ks), 1.0)
    ev = oracle.quantize_e4m3_np(nv.float().numpy() * np.float32(1 / vs), 1.0)
    got_k = kc.view(torch.uint8).view(-1, Hkv, 128).cpu().numpy()
    got_v = vc.view(torch.uint8).view(-1, Hkv, 128).cpu().numpy()
    assert np.array_equal(got_k[slots[keep].numpy()], ek[keep.numpy()])
    assert np.array_equal(got_v[slots[keep].numpy()], ev[keep.numpy()])
    untouched = np.ones(NB * bs, dtype=bool)
    untouched[slots[keep].numpy()] = False
    assert not got_k[untouched].any()


def test_append_then_decode_fp8():
    lens = [40, 513]
    d = W.make_decode(dict(W.C2, batch_size=2, seq_len=513, kv_dtype="fp8_e4m3"), device="cuda", lens=lens,
                      extra_blocks=2)
    g = torch.Generator().manual_seed(9)
    nk, nv = ((torch.randn(2, 8, 128, generator=g)).bfloat16().to(DEV) for _ in range(2))
    bs = 16
    slots = torch.tensor([int(d.block_table[b, (lens[b] - 1) // bs]) * bs + (lens[b] - 1) % bs for b in range(2)],
                         device=DEV)
    A.cache_append(nk, nv, d.k_cache, d.v_cache, slots, k_scale=d.k_scale, v_scale=d.v_scale)
    out = A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
    ref = oracle.decode_fp8_np(d.q.cpu(), d.k_cache.cpu(), d.v_cache.cpu(), d.block_table.cpu(), d.seq_lens.cpu(),
                               d.k_scale, d.v_scale)
    base = sdpa_decode_bf16(d.q, (d.k_cache.float() * d.k_scale).bfloat16(), (d.v_cache.float() * d.v_scale).bfloat16(),
                            d.block_table, d.seq_lens)
    check("append+decode fp8", out, ref, base)


# ------------------------------------------------------------------ runner on the GPU
def test_runner_b200_backend_end_to_end():
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    p = subprocess.Popen([sys.executable, "-m", "paper_2505_03780_b200.runner", "--binding",
                          str(ROOT / "paper_2505_03780_b200/spaces/prefill.binding.json"), "--protocol", "1"],
                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True, env=env, cwd=ROOT)

    def ask(m):
        p.stdin.write(json.dumps(m) + "\n")
        p.stdin.flush()
        return json.loads(p.stdout.readline())

    hello = ask({"type": "hello", "protocol": 1})
    assert "B200" in hello["fingerprint"]["device_name"] and "graph-timing" in hello["capabilities"]
    shape = dict(W.C1)
    ok = ask({"type": "evaluate", "config": pcfg(), "shape": shape, "warmups": 2, "reps": 5})
    assert ok["status"] == "ok" and len(ok["latencies_ms"]) == 5 and ok["compile_ms"] > 0
    bad = ask({"type": "evaluate", "config": pcfg(bm=64, bn=64), "shape": shape, "warmups": 1, "reps": 2})
    assert bad["status"] == "invalid" and "BLOCK_M" in bad["reason"]
    p.stdin.write(json.dumps({"type": "shutdown"}) + "\n")
    p.stdin.flush()
    assert p.wait(timeout=30) == 0


def test_decode_flat_fused_merge_option(tmp_path):
    """The in-kernel merge (B200ATTN_FLAT_MERGE=1, read once per process -> a subprocess): 64 ragged
    sequences split across 2-3 CTAs each, merged by the CTA finishing their last piece; vs the oracle."""
    script = tmp_path / "fused.py"
    script.write_text(
        "import sys, torch\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "from paper_2505_03780_b200 import attention as A, workload as W\n"
        "g = torch.Generator().manual_seed(21)\n"
        "lens = torch.randint(1, 3000, (64,), generator=g).tolist(); lens[3] = 0\n"
        "d = W.make_decode(dict(W.C2, batch_size=64, seq_len=max(lens)), device='cpu', lens=lens, extra_blocks=4)\n"
        "args = [t.cuda() for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]\n"
        "p = A.DecodePlan(*args, config=dict(num_splits=0, num_stages=4, TILE_N=16))\n"
        "assert p.kernels_per_run() == 1, p.kernels_per_run()\n"
        f"torch.save(dict(out=p.run().cpu(), lens=lens), {str(tmp_path / 'out.pt')!r})\n")
    env = dict(os.environ, B200ATTN_FLAT_MERGE="1")
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = torch.load(tmp_path / "out.pt")
    lens = res["lens"]
    d = W.make_decode(dict(W.C2, batch_size=64, seq_len=max(lens)), device="cpu", lens=lens, extra_blocks=4)
    assert res["out"][3].abs().max().item() == 0
    sub = [0, 1, 2, 40, 63]
    ref = oracle.decode(d.q[sub], d.k_cache, d.v_cache, d.block_table[sub], d.seq_lens[sub])
    args = [t.to(DEV) for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
    ki = torch.tensor(sub, device=DEV)
    check("decode flat fused in-kernel merge", res["out"][sub], ref,
          sdpa_decode_bf16(args[0][ki], args[1], args[2], args[3][ki], args[4][ki]))


@pytest.mark.parametrize("band", [1, 2, 3])
def test_prefill_banded_order_forced(tmp_path, band):
    """The L2-aware banded work order (on by default only above ~64 MB of K/V) forced onto small
    problems with tiny bands (B200ATTN_PREFILL_BAND, read once per process -> a subprocess): varlen
    (schedule kernel) and single-sequence (analytic) item decoding, causal and not, GQA 4 and 8,
    BLOCK_M 128/256 and the CTA pair; every case vs the oracle."""
    cases = [([300, 77, 1000, 129, 1], 32, 8, True, pcfg()), ([1000], 32, 8, True, pcfg()),
             ([700] * 3, 32, 8, True, pcfg()), ([520] * 4, 16, 2, False, pcfg(128, 128, 3)),
             ([700, 129], 16, 2, True, pcfg(128, 128, 2)), ([900], 16, 2, False, pcfg(128, 128, 3)),
             ([500, 1, 640], 32, 8, False, pcfg()), ([1000, 260], 32, 4, True, pcfg(256, 128, 2, pair=True)),
             ([1100], 32, 4, True, pcfg(256, 128, 2, pair=True))]
    script = tmp_path / "banded.py"
    script.write_text(
        "import sys, json, torch, numpy as np\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "from paper_2505_03780_b200 import attention as A\n"
        f"cases = json.loads({json.dumps(json.dumps(cases))})\n"
        "outs = []\n"
        "for i, (lens, hq, hkv, causal, cfg) in enumerate(cases):\n"
        "    g = torch.Generator().manual_seed(100 + i)\n"
        "    T = sum(lens)\n"
        "    q, k, v = (torch.randn(T, h, 128, generator=g).bfloat16().cuda() for h in (hq, hkv, hkv))\n"
        "    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32).cuda()\n"
        "    outs.append(A.prefill_varlen(q, k, v, cu, max(lens), causal=causal, config=cfg).cpu())\n"
        f"torch.save(outs, {str(tmp_path / 'out.pt')!r})\n")
    env = dict(os.environ, B200ATTN_PREFILL_BAND=str(band))
    r = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    outs = torch.load(tmp_path / "out.pt")
    for i, (lens, hq, hkv, causal, cfg) in enumerate(cases):
        g = torch.Generator().manual_seed(100 + i)
        T = sum(lens)
        q, k, v = (torch.randn(T, h, 128, generator=g).bfloat16() for h in (hq, hkv, hkv))
        cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
        ref = oracle.prefill(q, k, v, cu, causal=causal)
        base = sdpa_prefill_bf16(q.to(DEV), k.to(DEV), v.to(DEV), cu, causal)
        check(f"prefill banded order band={band} {lens} {hq}/{hkv} causal={causal}"
              f"{' pair' if cfg['waves_per_eu'] == 2 else ''}", outs[i], ref, base)


def test_prefill_1x16k_banded_default():
    """One 16k-token sequence (K/V 67 MB: the banded order is on by default): every q head of 4
    spread q blocks vs the oracle (rows are independent)."""
    x = W.make_prefill(dict(W.C1, seq_len=16384), device="cpu")
    qd, kd, vd, cud = x.q.to(DEV), x.k.to(DEV), x.v.to(DEV), x.cu_seqlens.to(DEV)
    out = A.prefill_varlen(qd, kd, vd, cud, x.max_seqlen).cpu()
    for a in (0, 5000, 12000, 16384 - 32):  # causal: rows up to a+31 see keys [0, a+32)
        sl = slice(0, a + 32)
        cu = torch.tensor([0, a + 32], dtype=torch.int32)
        ref = oracle.prefill_blas(x.q[sl], x.k[sl], x.v[sl], cu)
        base = sdpa_prefill_bf16(qd[sl], kd[sl], vd[sl], cu, True)
        check(f"1x16k banded rows {a}..{a + 31}", out[a:a + 32], ref[a:a + 32], base[a:a + 32])
