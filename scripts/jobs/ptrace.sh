# K1 per-CTA launch timelines (trace library): span of a launch and the gap to the previous one
export PYTHONPATH=$PWD
L=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so
O=gpurun_out/${1:-pt}
for pdl in 1 0; do
  B200ATTN_PDL=$pdl B200ATTN_LIB=$L timeout 300 python scripts/perf.py ptrace --shapes C1,C3,1x16k --tag "pdl$pdl"
  B200ATTN_PDL=$pdl B200ATTN_LIB=$L timeout 300 python scripts/perf.py ptrace --shapes C1 --tag "pdl$pdl-bm128ns3" \
    --cfg '{"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1, "PRE_LOAD_V": false}'
done > ${O}_ptrace.log 2>&1
