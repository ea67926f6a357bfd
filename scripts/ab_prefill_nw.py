"""A/B prefill softmax layouts: num_warps 4 (one thread per S row) vs 8 (two threads per row),
graph-replayed, on C3 / 1x16k / C1."""
import sys, torch
from paper_2505_03780_b200 import attention as A, workload as W


def run(x, cfg, reps):
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
    p.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): p.run()
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / reps)
    return best, x.flops / best / 1e9


def cfg(bm, ns, nw):
    return dict(BLOCK_M=bm, BLOCK_N=128, num_warps=nw, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)


for name, shape, reps in (("C3", W.C3, 10), ("1x16k", dict(W.C1, seq_len=16384), 10), ("C1", W.C1, 100),
                          ("4x2k", dict(W.C1, batch_size=4, seq_len=2048), 20)):
    x = W.make_prefill(shape, device="cuda")
    for bm in (256, 128):
        for ns in (1, 2):
            for nw in (4, 8):
                ms, tf = run(x, cfg(bm, ns, nw), reps)
                print(f"{name} BM{bm} ns{ns} nw{nw}: {ms*1e3:8.1f} us {tf:7.1f} TFLOP/s", flush=True)
