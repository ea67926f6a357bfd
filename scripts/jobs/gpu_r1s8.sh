set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for kv in bfloat16 fp8_e4m3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_flat -s 3 -c 1 -o gpurun_out/dec_${kv}_r1s8 python -c "
import torch
from paper_2505_03780_b200 import attention as A, workload as W
d = W.make_decode(dict(W.C2, kv_dtype='$kv'), device='cuda')
for _ in range(5): A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
torch.cuda.synchronize()
" > gpurun_out/r1s8_ncu_$kv.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
