# EARLY S release needs K_{j+1} resident during step j: A/B at num_stages 3 and 4
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for ns in 2 3 4; do
C="{\"BLOCK_M\": 256, \"BLOCK_N\": 128, \"num_warps\": 4, \"num_stages\": $ns, \"waves_per_eu\": 1, \"PRE_LOAD_V\": false}"
PREFILL_CFG="$C" timeout 200 python scripts/ab_prefill.py 2>&1 | grep -v C1 | sed "s/^/early1 ns$ns /"
PREFILL_CFG="$C" B200ATTN_LIB=_ab/lib_early0.so timeout 200 python scripts/ab_prefill.py 2>&1 | grep -v C1 | sed "s/^/early0 ns$ns /"
done > gpurun_out/r1s52_ab.txt
cat gpurun_out/r1s52_ab.txt
