export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fp8 or golden or decode" 2>&1 | tail -6
timeout 300 python scripts/perf_decode_small.py 2>&1
