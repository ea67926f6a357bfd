set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1s7_pytest.log
B200ATTN_FP8_HWCVT=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8 or decode" 2>&1 | tail -2 >> gpurun_out/r1s7_pytest.log
timeout 300 python scripts/perf_decode_small.py > gpurun_out/r1s7_dec.log 2>&1
timeout 300 python scripts/perf_decode.py > gpurun_out/r1s7_dec_c2c4.log 2>&1
cat gpurun_out/r1s7_pytest.log gpurun_out/r1s7_dec.log gpurun_out/r1s7_dec_c2c4.log
