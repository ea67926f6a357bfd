export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or golden" 2>&1 | tail -3
for v in 0 1 0 1; do B200ATTN_PREFILL_SPECULATE=$v TAG=spec$v timeout 300 python scripts/ab_prefill.py 2>&1; done
