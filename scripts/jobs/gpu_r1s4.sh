set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
# trace-enabled build (separate .so; the product library is untouched)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_TRACE -o /tmp/libtrace.so paper_2505_03780_b200/csrc/capi.cu > gpurun_out/r1s4_tracebuild.log 2>&1
for v in 1 0; do
  B200ATTN_PREFILL_TWOPASS=$v timeout 300 python scripts/ab_prefill.py >> gpurun_out/r1s4_ab.log 2>&1
  B200ATTN_PREFILL_TWOPASS=$v B200ATTN_LIB=/tmp/libtrace.so timeout 300 python scripts/trace_prefill.py > gpurun_out/r1s4_trace_tp$v.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_flat -s 3 -c 1 -o gpurun_out/dec_fp8_r1s4 python -c "
import torch
from paper_2505_03780_b200 import attention as A, workload as W
d = W.make_decode(dict(W.C2, kv_dtype='fp8_e4m3'), device='cuda')
for _ in range(5): A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
torch.cuda.synchronize()
" > gpurun_out/r1s4_ncu_fp8.log 2>&1
cat gpurun_out/r1s4_ab.log; head -30 gpurun_out/r1s4_trace_tp1.log; head -30 gpurun_out/r1s4_trace_tp0.log
