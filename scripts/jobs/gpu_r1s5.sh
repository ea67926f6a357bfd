set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/r1s5_pytest.log
B200ATTN_PREFILL_WPR=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or golden" 2>&1 | tail -3 >> gpurun_out/r1s5_pytest.log
for v in 1 2; do B200ATTN_PREFILL_WPR=$v timeout 300 python scripts/ab_prefill.py 2>&1 | sed "s/^/wpr$v /" >> gpurun_out/r1s5_ab.log; done
for v in 0 1; do B200ATTN_FP8_HWCVT=$v timeout 300 python scripts/perf_decode_small.py 2>&1 | grep fp8 | sed "s/^/hw$v /" >> gpurun_out/r1s5_fp8.log; done
B200ATTN_FP8_HWCVT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8" 2>&1 | tail -3 >> gpurun_out/r1s5_pytest.log
cat gpurun_out/r1s5_pytest.log gpurun_out/r1s5_ab.log gpurun_out/r1s5_fp8.log
