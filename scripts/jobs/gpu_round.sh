set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r1s2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s2_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s2_bench.json 2> gpurun_out/r1s2_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1s2_bench_ref.json 2>&1
timeout 600 python bench.py --workload prefill > gpurun_out/r1s2_bench_prefill.json 2>&1
cat gpurun_out/r1s2_pytest.log gpurun_out/r1s2_smoke.log gpurun_out/r1s2_bench.json gpurun_out/r1s2_bench_ref.json gpurun_out/r1s2_bench_prefill.json
