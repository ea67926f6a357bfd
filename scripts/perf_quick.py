"""Quick device-time sweep of the BASELINE configs (CUDA events, L2 flushed between reps)."""
import sys, json
import torch
from paper_2505_03780_b200 import attention as A, workload as W

dev = "cuda"
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

def timeit(fn, reps=10, warm=3, do_flush=True):
    for _ in range(warm): fn()
    ts = []
    for _ in range(reps):
        if do_flush: flush.zero_()
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort(); return ts[len(ts)//2]

def pf(shape, cfg):
    x = W.make_prefill(shape, device=dev)
    out = torch.empty_like(x.q)
    f = lambda: A.prefill_varlen(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, out=out, config=cfg)
    ms = timeit(f)
    return ms, x.flops / ms / 1e9

cfgs = []
for bm in (128, 256):
    for bn in (64, 128):
        for ns in (2, 3, 4):
            cfgs.append(dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=4, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False))
for name, shape in (("C1", W.C1), ("C3", W.C3)):
    for cfg in cfgs:
        try:
            ms, tf = pf(shape, cfg)
            print(f"{name} {cfg['BLOCK_M']}/{cfg['BLOCK_N']}/{cfg['num_stages']}: {ms*1e3:.1f} us  {tf:.1f} TFLOP/s", flush=True)
        except Exception as e:
            print(name, cfg['BLOCK_M'], cfg['BLOCK_N'], cfg['num_stages'], "ERR", str(e)[:80])

def dec(shape, cfg):
    d = W.make_decode(shape, device=dev)
    out = torch.empty_like(d.q)
    f = lambda: A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, out=out, config=cfg)
    ms = timeit(f)
    return ms, d.kv_bytes / ms / 1e6, A.decode_num_splits(tuple(d.q.shape), tuple(d.k_cache.shape), d.block_table.shape[1], d.max_seq_len, cfg)

C4s = dict(W.C4, batch_size=32)  # one GPU's shard at W=8
for name, shape in (("C2", W.C2), ("C4/8", C4s)):
    for ns in (2, 3, 4, 6):
        for sp in (0, 1, 2, 4, 8):
            cfg = dict(num_splits=sp, num_stages=ns, TILE_N=128)
            try:
                ms, gbs, s = dec(shape, cfg)
                print(f"{name} ns{ns} splits{sp}->{s}: {ms*1e3:.1f} us  {gbs:.0f} GB/s", flush=True)
            except Exception as e:
                print(name, ns, sp, "ERR", str(e)[:100])
