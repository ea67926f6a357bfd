export PYTHONPATH=$PWD
mkdir -p gpurun_out
C='{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'
timeout 900 python -m pytest tests -q -m gpu -k "decode or flat or combine or step" > gpurun_out/r2z_tests.log 2>&1; tail -6 gpurun_out/r2z_tests.log
timeout 300 python scripts/perf.py time --tag k3new --shapes d1x2k,d1x8k,d4x2k,d16x512,d64x512,C2,C4shard,C2fp8,b1x32k --cfg "$C" > gpurun_out/r2z_time.log 2>&1
timeout 300 python scripts/perf.py time --tag dispatch --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x128,d16x512,d64x512,C2 >> gpurun_out/r2z_time.log 2>&1
cat gpurun_out/r2z_time.log
