# PDL between K2' and K3': decode parity, then bench A/B (B200ATTN_PDL=1 vs 0)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "decode or append or fp8" 2>&1 | tail -3 > gpurun_out/r1s55_pytest.log
cat gpurun_out/r1s55_pytest.log
for rep in 1 2; do
for pdl in 1 0; do
B200ATTN_PDL=$pdl timeout 300 python bench.py --no-extra --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl$pdl', round(d['value'],1), round(d['ms_per_step']*1e3,2), 'us  e2e', round(d['e2e']['value'],1), 'kernel', round(d['roofline']['achieved'],1))"
done; done > gpurun_out/r1s55_ab.txt 2>&1
cat gpurun_out/r1s55_ab.txt
