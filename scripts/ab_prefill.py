"""A/B the prefill softmax variants (env B200ATTN_PREFILL_TWOPASS) on C3 / long / C1 (graph replay)."""
import json, os, sys, torch
from paper_2505_03780_b200 import attention as A, workload as W

CFG = json.loads(os.environ["PREFILL_CFG"]) if os.environ.get("PREFILL_CFG") else None


def run(shape, reps=20, cfg=None):
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

tag = os.environ.get("TAG", "prefill")
for name, shape in (("C3", W.C3), ("1x16k", dict(W.C1, seq_len=16384)), ("C1", W.C1)):
    ms, tf = run(shape, reps=20 if name != "C1" else 200, cfg=CFG if name != "C1" else None)
    print(f"{tag} {name}: {ms*1e3:.1f} us {tf:.1f} TFLOP/s", flush=True)
