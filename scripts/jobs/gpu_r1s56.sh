# e2e through DecodePlan vs one-shot paged_decode
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for rep in 1 2; do
timeout 300 python bench.py --no-extra --no-cpu-baseline 2>gpurun_out/r1s56_err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print('value', round(d['value'],1), 'e2e plan', round(e['value'],1), round(e['ms_per_step']*1e3,1), 'us  one-shot', round(e['one_shot']['value'],1), round(e['one_shot']['ms_per_step']*1e3,1), 'us')"
done > gpurun_out/r1s56_ab.txt 2>&1
tail -3 gpurun_out/r1s56_err.txt >> gpurun_out/r1s56_ab.txt
cat gpurun_out/r1s56_ab.txt
