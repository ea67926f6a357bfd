export PYTHONPATH=$PWD
mkdir -p gpurun_out
C='{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'
B200ATTN_LIB=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so timeout 600 python scripts/perf.py dtrace --shapes d1x128,d1x2k,d1x8k,d16x512,d4x2k,d64x512 --cfg "$C" > gpurun_out/r2w_dtrace.log 2>&1
timeout 600 python scripts/perf.py time --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x128,d16x512,d64x512 > gpurun_out/r2w_time.log 2>&1
timeout 600 python scripts/perf.py time --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x128,d16x512,d64x512 --cfg "$C" --tag flat >> gpurun_out/r2w_time.log 2>&1
timeout 600 python scripts/perf.py e2e > gpurun_out/r2w_e2e.log 2>&1
cat gpurun_out/r2w_dtrace.log gpurun_out/r2w_time.log gpurun_out/r2w_e2e.log
