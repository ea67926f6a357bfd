import torch
from paper_2505_03780_b200 import attention as A, workload as W
def run(shape, cfg=None, reps=5):
    x = W.make_prefill(shape, device="cuda")
    p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg, causal=shape.get("causal", True))
    p.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): p.run()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); g.replay(); e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return ms, x.flops / ms / 1e9
for name, shape in [("C3", W.C3), ("4x8192 causal", dict(W.C1, batch_size=4, seq_len=8192)),
                    ("1x16384 causal", dict(W.C1, batch_size=1, seq_len=16384)),
                    ("16x2048 causal", dict(W.C1, batch_size=16, seq_len=2048)),
                    ("4x8192 noncausal", dict(W.C1, batch_size=4, seq_len=8192, causal=False)),
                    ("64x512 causal", dict(W.C1, batch_size=64, seq_len=512))]:
    ms, tf = run(shape)
    print(f"{name}: {ms*1e3:.1f} us {tf:.1f} TFLOP/s", flush=True)
