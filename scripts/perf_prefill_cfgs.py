"""Every compiled prefill variant on C3, 1 x 16k and C1 (graph replay)."""
import sys, torch
from paper_2505_03780_b200 import attention as A, workload as W


def run(x, cfg, reps):
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
    p.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            p.run()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return ms, x.flops / ms / 1e9


for name, shape, reps in (("C3", W.C3, 10), ("1x16k", dict(W.C1, seq_len=16384), 10), ("C1", W.C1, 100)):
    x = W.make_prefill(shape, device="cuda")
    for bm in (256, 128):
        for bn in (128, 64):
            for ns in (1, 2, 3, 4):
                cfg = dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=4, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
                try:
                    ms, tf = run(x, cfg, reps)
                    print(f"{name} BM{bm} BN{bn} ns{ns}: {ms*1e3:8.1f} us {tf:7.1f} TFLOP/s", flush=True)
                except Exception as ex:
                    print(name, bm, bn, ns, "ERR", str(ex)[:100], flush=True)
