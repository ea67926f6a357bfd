export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "jumps" 2>&1 | grep -E "parity|Error|assert|passed|failed" | head -20
B200ATTN_PREFILL_SPECULATE=0 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "jumps" 2>&1 | grep -E "parity|Error|assert|passed|failed" | head -20
