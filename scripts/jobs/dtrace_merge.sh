C='{"TILE_N": 16, "num_splits": 0, "num_stages": 5}'
for v in "B200ATTN_FLAT_MERGE=0"; do
  env $v B200ATTN_LIB=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so timeout 300 python scripts/perf.py dtrace --shapes C2,C4shard --cfg "$C" --tag "$v" --per-cta
done > gpurun_out/r2j_dtrace.log 2>&1
