export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefill or golden" 2>&1 | tail -2
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -o /tmp/lib_base.so _ab_base/csrc/capi.cu > /tmp/base_build.log 2>&1; tail -2 /tmp/base_build.log
echo "== base (no TMEM-load pipelining)"
for CFG in '{"BLOCK_M":256,"BLOCK_N":128,"num_warps":4,"num_stages":2,"waves_per_eu":1,"PRE_LOAD_V":false}' '{"BLOCK_M":128,"BLOCK_N":128,"num_warps":4,"num_stages":3,"waves_per_eu":1,"PRE_LOAD_V":false}'; do B200ATTN_LIB=/tmp/lib_base.so TAG=base PREFILL_CFG=$CFG timeout 300 python scripts/ab_prefill.py 2>&1; done
for E in 3 0 2 4; do
  L=/tmp/lib_e$E.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_PREFILL_EMU=$E -o $L paper_2505_03780_b200/csrc/capi.cu > /dev/null 2>&1
  echo "== EMU $E"
  for CFG in '{"BLOCK_M":256,"BLOCK_N":128,"num_warps":4,"num_stages":2,"waves_per_eu":1,"PRE_LOAD_V":false}' '{"BLOCK_M":128,"BLOCK_N":128,"num_warps":4,"num_stages":3,"waves_per_eu":1,"PRE_LOAD_V":false}'; do B200ATTN_LIB=$L TAG=e$E PREFILL_CFG=$CFG timeout 300 python scripts/ab_prefill.py 2>&1; done
done
