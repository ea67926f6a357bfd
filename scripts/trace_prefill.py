import ctypes, numpy as np, torch
from paper_2505_03780_b200 import attention as A, workload as W, _native
lib = _native.load()
x = W.make_prefill(dict(W.C1, batch_size=4, seq_len=8192), device="cuda")
p = A.PrefillPlan(x.q, x.k, x.v, x.cu_seqlens, x.max_seqlen)
for _ in range(3): p.run()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (16 * 512))()
lib.b200attn_debug_trace(buf, 16 * 512)
t = np.frombuffer(buf, dtype=np.uint64).reshape(16, 512).astype(np.int64)
base = t[0, 0]
n = 40
print("tile  S0   P0(sm0)  S1  P1  MMA-sees-P0 MMA-sees-P1 Vfull  QK0-issued (cycles rel. to S0 of tile)")
for j in range(1, n):
    r = t[:, j] - t[0, j]
    print(j, " ".join(f"{v:7d}" for v in r[:8]), "  dS0:", t[0, j] - t[0, j - 1],
          " | S seen w0-3:", " ".join(f"{v:6d}" for v in r[12:16]), " P done w0-3:", " ".join(f"{v:6d}" for v in r[8:12]))
