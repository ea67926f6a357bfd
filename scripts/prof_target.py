"""Small driver for ncu: runs one config a few times. usage: prof_target.py {decode|prefill} [cfg-json]"""
import sys, json
import torch
from paper_2505_03780_b200 import attention as A, workload as W
which = sys.argv[1]
cfg = json.loads(sys.argv[2]) if len(sys.argv) > 2 else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if which == "decode":
    d = W.make_decode(W.C2, device="cuda")
    out = torch.empty_like(d.q)
    for _ in range(n):
        A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, max_seq_len=d.max_seq_len, out=out, config=cfg)
else:
    shape = W.C3 if which == "prefill" else W.C1
    x = W.make_prefill(shape, device="cuda")
    out = torch.empty_like(x.q)
    for _ in range(n):
        A.prefill_varlen(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, out=out, config=cfg)
torch.cuda.synchronize()
print("done")
