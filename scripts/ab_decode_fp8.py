"""A/B the fp8-cache decode ring depth (num_stages) on C2 and 256 x 8192, graph-replayed."""
import torch
from paper_2505_03780_b200 import attention as A, workload as W


def run(d, ns, reps=20):
    cfg = {"num_splits": 0, "num_stages": ns, "TILE_N": 16}
    p = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, config=cfg,
                     k_scale=d.k_scale, v_scale=d.v_scale)
    p.run(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): p.run()
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); g.replay(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / reps)
    return best


for name, shape in (("C2", dict(W.C2, kv_dtype="fp8_e4m3")), ("256x8192", dict(W.C2, batch_size=256, seq_len=8192, kv_dtype="fp8_e4m3"))):
    d = W.make_decode(shape, device="cuda")
    for ns in (6, 8, 10, 8, 10):
        ms = run(d, ns)
        print(f"{name} fp8 ns{ns}: {ms*1e3:.1f} us {d.kv_bytes / ms / 1e6:.0f} GB/s", flush=True)
