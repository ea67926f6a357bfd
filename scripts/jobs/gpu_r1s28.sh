export PYTHONPATH=$PWD
for E in 3 0 4 2 3; do
  L=/tmp/lib_e$E.so
  [ -f $L ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_PREFILL_EMU=$E -o $L paper_2505_03780_b200/csrc/capi.cu > /dev/null 2>&1
  B200ATTN_LIB=$L timeout 300 python bench.py --workload prefill --steps 500 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('EMU $E bench prefill', round(d['value'],1), d['config']['variant']['BLOCK_M'], d['config']['variant']['num_stages'], d['clocks'])"
  B200ATTN_LIB=$L TAG=e$E PREFILL_CFG='{"BLOCK_M":256,"BLOCK_N":128,"num_warps":4,"num_stages":2,"waves_per_eu":1,"PRE_LOAD_V":false}' timeout 300 python scripts/ab_prefill.py 2>&1 | head -2
done
