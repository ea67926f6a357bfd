# one gpurun call: prefill ncu evidence + the full C5 sweep (ktune tune, exhaustive)
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s2_launches_prefill.csv python bench.py --workload prefill --steps 5 --warmup 3 > gpurun_out/r1s2_ncu_bench_prefill.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 -o gpurun_out/pf_r1s2 python scripts/prof_target.py prefill > gpurun_out/r1s2_ncu_pf.log 2>&1
timeout 3000 python scripts/c5_sweep.py run --out gpurun_out/c5 > gpurun_out/c5_run.log 2>&1
rm -rf gpurun_out/c5/cache
tail -5 gpurun_out/c5_run.log
