set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1s6_pytest.log
B200ATTN_FP8_HWCVT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8" 2>&1 | tail -2 >> gpurun_out/r1s6_pytest.log
for v in 0 1; do B200ATTN_FP8_HWCVT=$v timeout 300 python scripts/perf_decode_small.py 2>&1 | sed "s/^/hw$v /" >> gpurun_out/r1s6_fp8.log; done
timeout 300 python scripts/ab_prefill.py > gpurun_out/r1s6_ab.log 2>&1
cat gpurun_out/r1s6_pytest.log gpurun_out/r1s6_fp8.log gpurun_out/r1s6_ab.log
