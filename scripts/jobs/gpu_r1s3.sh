set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r1s3_pytest.log
timeout 300 python scripts/perf_decode_small.py > gpurun_out/r1s3_decode_small.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s3_bench.json 2> gpurun_out/r1s3_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 -o gpurun_out/pf_r1s3 python scripts/prof_target.py prefill > gpurun_out/r1s3_ncu_pf.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s3_launches_prefill.csv python scripts/prof_target.py prefill > /dev/null 2>&1
cat gpurun_out/r1s3_pytest.log gpurun_out/r1s3_decode_small.log gpurun_out/r1s3_bench.json
