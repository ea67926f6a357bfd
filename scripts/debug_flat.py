import sys; sys.path.insert(0, "oracle")
import numpy as np, torch, oracle
from paper_2505_03780_b200 import attention as A, workload as W
lens = [128]
d = W.make_decode(dict(W.C2, batch_size=1, seq_len=128), device="cpu", lens=lens, extra_blocks=3)
args = [t.cuda() for t in (d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)]
plan = A.DecodePlan(*args, config=dict(num_splits=0, num_stages=4, TILE_N=16))
plan.run_partial(); torch.cuda.synchronize()
ws = plan.ws.view(torch.float32)
C = 148; B = 1; NQ = 32; slots = C + B
po = ws[: slots * NQ * 128].view(slots, NQ, 128).cpu().numpy()
pml = ws[slots * NQ * 128: slots * NQ * 130].view(slots, NQ, 2).cpu().numpy()
cu = ws.view(torch.int32)[slots * NQ * 130: slots * NQ * 130 + 2].cpu().numpy()
print("cu", cu)
q = oracle.bf16_bits_to_f64(oracle.as_bf16_bits(d.q))[0]            # [32,128]
kc = oracle.bf16_bits_to_f64(oracle.as_bf16_bits(d.k_cache)); vc = oracle.bf16_bits_to_f64(oracle.as_bf16_bits(d.v_cache))
bt = d.block_table.numpy()[0]
for tile in range(8):
    c = int(((tile + 1) * C - 1) // 8); slot = c + 0
    K = kc[bt[tile]]; V = vc[bt[tile]]   # [16, 8, 128]
    s = np.einsum("hd,thd->ht", q, np.repeat(K, 4, axis=1)) / np.sqrt(128) * np.log2(np.e)
    m = s.max(1); p = np.exp2(s - m[:, None]); l = p.sum(1); o = np.einsum("ht,thd->hd", p, np.repeat(V, 4, axis=1))
    print(tile, "cta", c, "m err", np.abs(pml[slot, :, 0] - m).max(), "l err", np.abs(pml[slot, :, 1] - l).max(),
          "o err", np.abs(po[slot] - o).max(), "o|", np.abs(o).max(), "l", l[:3], pml[slot, :3, 1])
out = plan.run(); torch.cuda.synchronize()
ref = oracle.decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens)
print("final err", np.abs(out.float().cpu().numpy() - ref).max())
for rep in range(5):
    o2 = A.paged_decode(*args, config=dict(num_splits=0, num_stages=4, TILE_N=16)); torch.cuda.synchronize()
    print("paged_decode err", np.abs(o2.float().cpu().numpy() - ref).max())
