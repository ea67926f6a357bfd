export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or golden" 2>&1 | tail -3
timeout 600 python scripts/perf_prefill_cfgs.py 2>&1
