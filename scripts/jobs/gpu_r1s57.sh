# end-of-session evidence (session 3): tests, smoke, bench lines, reference arm, ncu launch lists + full captures
set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r1s57_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s57_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s57_bench.json 2> gpurun_out/r1s57_bench.err
timeout 600 python bench.py --workload prefill > gpurun_out/r1s57_bench_prefill.json 2> gpurun_out/r1s57_bench_prefill.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r1s57_bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s57_launches_prefill.csv python bench.py --workload prefill --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s57_launches_decode.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 -o gpurun_out/pf_r1s57 python scripts/prof_target.py prefill > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_flat -s 3 -c 1 -o gpurun_out/dec_r1s57 python scripts/prof_target.py decode null 6 > /dev/null 2>&1
cat gpurun_out/r1s57_pytest.log gpurun_out/r1s57_smoke.log
