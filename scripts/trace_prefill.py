"""clock64 trace of one steady-state prefill CTA (needs a -DB200_TRACE build via B200ATTN_LIB).
Config from argv: BLOCK_M num_stages num_warps (default: dispatch table)."""
import ctypes, sys, numpy as np, torch
from paper_2505_03780_b200 import attention as A, workload as W, _native
lib = _native.load()
cfg = None
if len(sys.argv) > 3:
    bm, ns, nw = map(int, sys.argv[1:4])
    cfg = dict(BLOCK_M=bm, BLOCK_N=128, num_warps=nw, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
x = W.make_prefill(dict(W.C1, batch_size=4, seq_len=8192), device="cuda")
p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen, config=cfg)
for _ in range(3): p.run()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (16 * 512))()
lib.b200attn_debug_trace(buf, 16 * 512)
t = np.frombuffer(buf, dtype=np.uint64).reshape(16, 512).astype(np.int64)
n = 40
print("config", cfg)
print("tile  S0   P0(sm0)  S1  P1  MMA-sees-P0 MMA-sees-P1 Vfull  QK0-issued (cycles rel. to S0 of tile)")
rows = []
for j in range(1, n):
    r = t[:, j] - t[0, j]
    rows.append(np.concatenate([r, [t[0, j] - t[0, j - 1]]]))
    print(j, " ".join(f"{v:7d}" for v in r[:8]), "  dS0:", t[0, j] - t[0, j - 1],
          " | S seen w0-3:", " ".join(f"{v:6d}" for v in r[12:16]), " P done w0-3:", " ".join(f"{v:6d}" for v in r[8:12]))
m = np.median(np.array(rows[5:]), axis=0)
print("median:", " ".join(f"{v:.0f}" for v in m))
