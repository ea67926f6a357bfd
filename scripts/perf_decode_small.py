"""Flat (TILE_N=16) vs split (TILE_N=128) decode across batch x context, bf16 and fp8 KV (graph replay)."""
import torch
from paper_2505_03780_b200 import attention as A, workload as W


def t(d, cfg, reps=50):
    p = A.DecodePlan(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, config=cfg,
                     k_scale=d.k_scale, v_scale=d.v_scale)
    p.run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(10):
            p.run()
    g.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 10 * 1e3


for kv in ("bfloat16", "fp8_e4m3"):
    for B, S in ((1, 128), (1, 4096), (1, 32768), (4, 2048), (16, 1024), (64, 4096), (256, 8192)):
        d = W.make_decode(dict(W.C2, batch_size=B, seq_len=S, kv_dtype=kv), device="cuda")
        row = [f"{kv:9s} B={B:4d} S={S:6d}"]
        for cfg in (dict(num_splits=0, num_stages=5 if kv == "bfloat16" else 8, TILE_N=16),
                    dict(num_splits=0, num_stages=4, TILE_N=128)):
            try:
                us = t(d, cfg)
                row.append(f"T{cfg['TILE_N']}: {us:8.1f} us {d.total_bytes / us / 1e3:7.0f} GB/s")
            except Exception as ex:
                row.append(f"T{cfg['TILE_N']}: {type(ex).__name__}")
        print(" | ".join(row), flush=True)
        del d
