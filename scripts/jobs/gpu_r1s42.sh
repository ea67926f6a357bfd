mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -5 > gpurun_out/r1s42_pytest.log
timeout 300 python scripts/ab_prefill_nw.py > gpurun_out/r1s42_ab.txt 2>&1
cat gpurun_out/r1s42_pytest.log gpurun_out/r1s42_ab.txt
