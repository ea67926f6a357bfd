set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r1s30_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s30_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s30_bench.json 2> gpurun_out/r1s30_bench.err
timeout 600 python bench.py --workload prefill > gpurun_out/r1s30_bench_prefill.json 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r1s30_bench_ref.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 -o gpurun_out/pf_r1s30 python scripts/prof_target.py prefill > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s30_launches_prefill.csv python bench.py --workload prefill --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s30_launches_decode.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
for kv in bfloat16 fp8_e4m3; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_flat -s 3 -c 1 -o gpurun_out/dec_${kv}_r1s30 python -c "
import torch
from paper_2505_03780_b200 import attention as A, workload as W
d = W.make_decode(dict(W.C2, kv_dtype='$kv'), device='cuda')
for _ in range(5): A.paged_decode(d.q, d.k_cache, d.v_cache, d.block_table, d.seq_lens, k_scale=d.k_scale, v_scale=d.v_scale)
torch.cuda.synchronize()
" > /dev/null 2>&1
done
cat gpurun_out/r1s30_pytest.log gpurun_out/r1s30_smoke.log
