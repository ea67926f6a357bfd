#!/usr/bin/env bash
# compute-sanitizer memcheck / racecheck / synccheck over small cases of every kernel (
# VERDICT r1 "sanitizer pass"): K1 prefill (1 and 2 q heads per CTA, 4 and 8 softmax warps per
# tile, causal + non-causal, varlen with the schedule kernel), K2' flat decode (bf16 + fp8 caches,
# fused in-kernel merge and the K3' combine path; Hkv = 1/2/4; batch > 1024), K2/K3 split decode, cache_append (+fp8),
# the three K3' launch shapes, and DecodeStep's zero-copy ingest kernel (bf16 + fp8).
# Usage: bash scripts/sanitize.sh OUT_PREFIX   -> OUT_PREFIX_{memcheck,racecheck,synccheck}.log
set -u
OUT=${1:-gpurun_out/sanitize}
export PYTHONPATH=$PWD
CASES=$(cat <<'EOF'
import sys, torch
sys.path.insert(0, "oracle")
from paper_2505_03780_b200 import attention as A, workload as W
def pf(lens, bm, nw, ns, causal=True, hq=8, hkv=2):
    x = W.make_prefill(dict(W.C1, batch_size=len(lens), seq_len=max(lens), num_q_heads=hq, num_kv_heads=hkv), device="cuda")
    import itertools
    x.cu_seqlens[:] = torch.tensor([0] + list(itertools.accumulate(lens)), dtype=torch.int32, device="cuda")
    T = sum(lens)
    q, k, v = x.q[:T].contiguous(), x.k[:T].contiguous(), x.v[:T].contiguous()
    cfg = dict(BLOCK_M=bm, BLOCK_N=128, num_warps=nw, num_stages=ns, waves_per_eu=1, PRE_LOAD_V=False)
    A.prefill_varlen(q, k, v, x.cu_seqlens, max(lens), causal=causal, config=cfg)
pf([300], 256, 4, 3); pf([300], 128, 4, 3); pf([200, 1, 129], 256, 8, 2); pf([200, 77], 128, 8, 1, causal=False)
for B, cfg in ((64, dict(num_splits=0, num_stages=4, TILE_N=16)), (3, dict(num_splits=0, num_stages=4, TILE_N=16)),
               (3, dict(num_splits=4, num_stages=4, TILE_N=128))):
    d = W.make_decode(dict(W.C2, batch_size=B, seq_len=200), device="cuda", lens=[200, 1, 77] * (B // 3) + [5] * (B % 3))
    A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=cfg)
    A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=cfg)
    nk = torch.randn(B, 8, 128, device="cuda").bfloat16()
    A.cache_append(nk, nk, d.k_cache, d.v_cache, torch.arange(B, device="cuda") * 3)
for hkv, bs in ((1, 16), (2, 32), (4, 16)):  # K2' at Hkv < 8 (PPT = 8 / Hkv page chunks per tile)
    d = W.make_decode(dict(W.C2, batch_size=4, seq_len=300, num_q_heads=8 * hkv, num_kv_heads=hkv, block_size=bs),
                      device="cuda", lens=[300, 1, 77, 129])
    A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=dict(num_splits=0, num_stages=4, TILE_N=16))
d = W.make_decode(dict(W.C2, batch_size=1100, seq_len=40), device="cuda", lens=[40, 1, 17] * 366 + [5, 5])
A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=dict(num_splits=0, num_stages=4, TILE_N=16))
f = W.make_decode(dict(W.C2, batch_size=3, seq_len=300, kv_dtype="fp8_e4m3"), device="cuda", lens=[300, 5, 64])
A.paged_decode(f.q, f.k_cache, f.v_cache, f.block_table, f.seq_lens, k_scale=f.k_scale, v_scale=f.v_scale)
nk = torch.randn(3, 8, 128, device="cuda").bfloat16()
A.cache_append(nk, nk, f.k_cache, f.v_cache, torch.arange(3, device="cuda"), k_scale=f.k_scale, v_scale=f.v_scale)
# K3' in its three shapes: (8 warps, 8 in flight) one CTA per SM, (8, 4), (4, 1) — 1 x 4000 (many pieces), 12 x 300
for B, ctx in ((1, 4000), (12, 300)):
    d = W.make_decode(dict(W.C2, batch_size=B, seq_len=ctx), device="cuda")
    A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, config=dict(num_splits=0, num_stages=4, TILE_N=16))
# DecodeStep's zero-copy path: the ingest kernel (PCIe reads of pinned host memory, copy + append, bf16 and
# fp8 caches) and K2'/K3' writing the output into pinned host memory
for kvd in ("bf16", "fp8_e4m3"):
    d = W.make_decode(dict(W.C2, batch_size=5, seq_len=300, kv_dtype=kvd), device="cuda", lens=[300, 1, 77, 129, 16],
                      extra_blocks=2)
    st = A.DecodeStep(d.k_cache, d.v_cache, d.block_table, batch=5, num_q_heads=32, k_scale=d.k_scale, v_scale=d.v_scale)
    bt = d.block_table.cpu()
    slots = torch.tensor([int(bt[b, (n - 1) // 16]) * 16 + (n - 1) % 16 for b, n in enumerate([300, 1, 77, 129, 16])])
    st.set_inputs(d.q.cpu(), torch.randn(5, 8, 128).bfloat16(), torch.randn(5, 8, 128).bfloat16(), slots, d.seq_lens.cpu())
    st(sync=True)
torch.cuda.synchronize()
print("sanitize cases done")
EOF
)
echo "$CASES" > /tmp/sanitize_cases.py
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 \
    python /tmp/sanitize_cases.py > ${OUT}_${tool}.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' ${OUT}_${tool}.log | tail -2)"
done
