# fp8-cache decode: ring depth 10 vs 8 (A/B), parity of the new variants
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 300 python scripts/ab_decode_fp8.py > gpurun_out/r1s58_ab.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "fp8" 2>&1 | tail -3 >> gpurun_out/r1s58_ab.txt
cat gpurun_out/r1s58_ab.txt
