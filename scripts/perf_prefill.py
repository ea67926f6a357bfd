import sys, torch
from paper_2505_03780_b200 import attention as A, workload as W
def run(shape, cfg, reps=10):
    x = W.make_prefill(shape, device="cuda")
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
    p.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): p.run()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return ms, x.flops / ms / 1e9
only = sys.argv[1] if len(sys.argv) > 1 else None
for name, shape in (("C3", W.C3), ("C1", W.C1)):
    for bm in (256, 128):
        for bn in (128, 64):
            for ns in (1, 2, 3, 4):
                cfg = dict(BLOCK_M=bm, BLOCK_N=bn, num_warps=4, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
                try:
                    ms, tf = run(shape, cfg)
                    print(f"{name} {bm}/{bn}/{ns}: {ms*1e3:.1f} us {tf:.1f} TFLOP/s", flush=True)
                except Exception as ex:
                    print(name, bm, bn, ns, "ERR", str(ex)[:120], flush=True)
