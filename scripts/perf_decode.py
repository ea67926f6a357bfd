import sys, torch
from paper_2505_03780_b200 import attention as A, workload as W
def run(shape, cfg, reps=20):
    d = W.make_decode(shape, device="cuda")
    p = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, config=cfg)
    g = torch.cuda.CUDAGraph(); p.run(); torch.cuda.synchronize()
    with torch.cuda.graph(g): p.run()
    gp = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gp): p.run_partial()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    res = []
    for gg in (g, gp):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): gg.replay()
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / reps
        res.append((ms, d.kv_bytes / ms / 1e6))
    return res
for name, shape in (("C2", W.C2), ("C4/8", dict(W.C4, batch_size=32))):
    for cfg in ([dict(num_splits=0, num_stages=ns, TILE_N=16) for ns in (3, 4, 5)] + [dict(num_splits=8, num_stages=4, TILE_N=128)]):
        try:
            (ms, gbs), (kms, kgbs) = run(shape, cfg)
            print(f"{name} {cfg}: total {ms*1e3:.1f} us {gbs:.0f} GB/s | K2 only {kms*1e3:.1f} us {kgbs:.0f} GB/s", flush=True)
        except Exception as ex:
            print(name, cfg, "ERR", str(ex)[:100])
