# prefill parity incl. the new num_warps=8 LSE / GQA / C3 cases
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "prefill" 2>&1 | tail -5 > gpurun_out/r1s54_pytest.log
cat gpurun_out/r1s54_pytest.log
