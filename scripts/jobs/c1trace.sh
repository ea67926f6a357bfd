# C1 (one 512-token sequence, 32 heads) first-item timeline of CTA 0 with the trace library
export PYTHONPATH=$PWD
L=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so
O=gpurun_out/${1:-c1t}
for pdl in 1 0; do
  for c in '{"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1, "PRE_LOAD_V": false}' \
           '{"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 8, "num_stages": 2, "waves_per_eu": 1, "PRE_LOAD_V": false}' \
           '{"BLOCK_M": 128, "BLOCK_N": 64, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1, "PRE_LOAD_V": false}'; do
    B200ATTN_PDL=$pdl B200ATTN_LIB=$L timeout 120 python scripts/perf.py c1trace --cfg "$c" --tag "pdl$pdl"
  done
done > ${O}_c1trace.log 2>&1
timeout 300 python scripts/perf.py single --shapes C1 >> ${O}_c1trace.log 2>&1
timeout 300 python scripts/perf.py time --op prefill --shapes C1 --all-variants >> ${O}_c1trace.log 2>&1
