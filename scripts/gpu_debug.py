"""First-contact GPU check: selftest + small prefill/decode parity, printing errors (no asserts)."""
import sys, time, traceback
sys.path.insert(0, "oracle")
import numpy as np, torch
import oracle
from paper_2505_03780_b200 import attention as A, workload as W

torch.manual_seed(0)
dev = "cuda"
print(torch.cuda.get_device_name(0), flush=True)

def run(name, fn):
    try:
        t = time.time(); r = fn(); torch.cuda.synchronize(); print(f"{name}: {r}  ({time.time()-t:.2f}s)", flush=True)
    except Exception as e:
        print(f"{name}: EXC {type(e).__name__}: {e}", flush=True); traceback.print_exc()

def st(mode):
    a = torch.randn(128, 128, device=dev).bfloat16(); b = torch.randn(16 if mode == 2 else 128, 128, device=dev).bfloat16()
    d = A.selftest_umma(mode, a, b)
    af, bf = a.float(), b.float()
    ref = af @ bf.t() if mode == 0 else (af @ bf if mode == 1 else af.t() @ bf.t())
    return float((d - ref).abs().max()), float(ref.abs().max())
for m in range(3): run(f"selftest{m}", lambda m=m: st(m))

def pf(lens, Hq=32, Hkv=8, causal=True, cfg=None):
    T = sum(lens); g = torch.Generator().manual_seed(1)
    q = torch.randn(T, Hq, 128, generator=g).bfloat16(); k = torch.randn(T, Hkv, 128, generator=g).bfloat16(); v = torch.randn(T, Hkv, 128, generator=g).bfloat16()
    cu = torch.tensor([0] + list(np.cumsum(lens)), dtype=torch.int32)
    ref = oracle.prefill(q, k, v, cu, causal=causal)
    out = A.prefill_varlen(q.to(dev), k.to(dev), v.to(dev), cu.to(dev), max(lens), causal=causal, config=cfg)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy()
    err = np.abs(o - ref)
    return f"maxabs={err.max():.3e} mean={err.mean():.2e} nan={np.isnan(o).sum()}"

run("prefill_128", lambda: pf([128]))
run("prefill_512", lambda: pf([512]))
run("prefill_200", lambda: pf([200]))
run("prefill_varlen", lambda: pf([1, 5, 127, 128, 129, 300]))
run("prefill_noncausal", lambda: pf([200, 64], causal=False))
run("prefill_mha_bm128", lambda: pf([300], Hq=8, Hkv=8, cfg=dict(BLOCK_M=128, BLOCK_N=128, num_warps=4, num_stages=3, waves_per_eu=1, PRE_LOAD_V=False)))
for bm in (128, 256):
    for bn in (64, 128):
        for ns in (2, 3, 4):
            cfg = dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=4, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
            run(f"prefill_cfg{bm}_{bn}_{ns}", lambda cfg=cfg: pf([300, 77], cfg=cfg))

def dec(lens, Hq=32, Hkv=8, bs=16, cfg=None):
    shape = dict(W.C2, batch_size=len(lens), seq_len=max(lens), num_q_heads=Hq, num_kv_heads=Hkv, block_size=bs)
    d = W.make_decode(shape, device="cpu", lens=lens, extra_blocks=3)
    ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
    out = A.paged_decode(d.q.to(dev), d.k_cache.to(dev), d.v_cache.to(dev), d.block_table.to(dev), d.seq_lens.to(dev), config=cfg)
    torch.cuda.synchronize()
    o = out.float().cpu().numpy(); err = np.abs(o - ref)
    return f"maxabs={err.max():.3e} mean={err.mean():.2e} nan={np.isnan(o).sum()}"

run("decode_single_tile", lambda: dec([128], cfg=dict(num_splits=1, num_stages=4, TILE_N=128)))
run("decode_4096_s1", lambda: dec([4096, 4096], cfg=dict(num_splits=1, num_stages=4, TILE_N=128)))
run("decode_ragged_s1", lambda: dec([1, 15, 16, 17, 127, 128, 129, 1000], cfg=dict(num_splits=1, num_stages=3, TILE_N=128)))
run("decode_ragged_s4", lambda: dec([1, 15, 16, 17, 127, 128, 129, 1000], cfg=dict(num_splits=4, num_stages=3, TILE_N=128)))
run("decode_auto", lambda: dec([4096] * 4))
run("decode_g8", lambda: dec([700, 3000], Hq=64, Hkv=8))
run("decode_bs32", lambda: dec([700, 3000], bs=32))
run("decode_bs64_s2", lambda: dec([700, 3000], bs=64, cfg=dict(num_splits=2, num_stages=2, TILE_N=128)))
for ns in (2, 3, 4, 5, 6):
    run(f"decode_ns{ns}", lambda ns=ns: dec([1000, 333], cfg=dict(num_splits=2, num_stages=ns, TILE_N=128)))
