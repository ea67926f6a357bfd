export PYTHONPATH=$PWD
mkdir -p gpurun_out
C='{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'
B200ATTN_LIB=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so timeout 600 python scripts/perf.py dtrace --shapes d1x128,d1x2k,d1x8k,d16x512,d4x2k,d64x512,C2 --cfg "$C" > gpurun_out/r2y_dtrace.log 2>&1
for v in 0 1; do B200ATTN_PDL_COMBINE=$v timeout 300 python scripts/perf.py time --tag pdlc$v --shapes d1x2k,d1x8k,d4x2k,d16x512,d64x512,C2 --cfg "$C"; done > gpurun_out/r2y_pdlc.log 2>&1
cat gpurun_out/r2y_dtrace.log gpurun_out/r2y_pdlc.log
