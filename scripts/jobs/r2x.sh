export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_api.py -q -m gpu -k "decode_step or mapped_ptr" > gpurun_out/r2x_tests.log 2>&1; tail -15 gpurun_out/r2x_tests.log
timeout 600 python scripts/perf.py e2e > gpurun_out/r2x_e2e.log 2>&1; cat gpurun_out/r2x_e2e.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-extra > gpurun_out/r2x_bench.json 2> gpurun_out/r2x_bench.err; cat gpurun_out/r2x_bench.json; tail -3 gpurun_out/r2x_bench.err
