export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python scripts/perf_decode.py 2>&1 | grep -v ERR
timeout 300 python scripts/perf_decode_small.py 2>&1 | grep -E "B=  64|B= 256|B=   1 S= 32768"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -o /tmp/lib_base.so _ab_base/csrc/capi.cu > /tmp/base_build.log 2>&1; tail -2 /tmp/base_build.log
for L in /tmp/lib_base.so $PWD/paper_2505_03780_b200/_lib/libb200attn.so /tmp/lib_base.so $PWD/paper_2505_03780_b200/_lib/libb200attn.so; do
  for CFG in '{"BLOCK_M":256,"BLOCK_N":128,"num_warps":4,"num_stages":2,"waves_per_eu":1,"PRE_LOAD_V":false}' '{"BLOCK_M":128,"BLOCK_N":128,"num_warps":4,"num_stages":3,"waves_per_eu":1,"PRE_LOAD_V":false}'; do
    B200ATTN_LIB=$L TAG=$(basename $L .so) PREFILL_CFG=$CFG timeout 300 python scripts/ab_prefill.py 2>&1
  done
done
