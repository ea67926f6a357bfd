export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "selftest" 2>&1 | tail -15
