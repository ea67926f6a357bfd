# per-config parity report (max-abs / max-rel vs the fp64 oracle, next to torch SDPA-bf16's own error)
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -v -s -k "golden or c1_full or c3_full or c2_full or c4_shard or fp8_c2 or gqa_shapes or score_jumps" 2>&1 | grep -oE "\[parity\].*|[0-9]+ passed.*|[0-9]+ failed.*" > gpurun_out/r1s60_parity.txt
cat gpurun_out/r1s60_parity.txt
