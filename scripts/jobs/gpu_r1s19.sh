export PYTHONPATH=$PWD
for H in 0 20000 1000000; do
  if [ $H = 0 ]; then L=$PWD/paper_2505_03780_b200/_lib/libb200attn.so; else
  L=/tmp/lib_h$H.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_WAIT_HINT_NS=$H -o $L paper_2505_03780_b200/csrc/capi.cu > /dev/null 2>&1; fi
  echo "== hint $H"
  B200ATTN_LIB=$L TAG=h$H timeout 300 python scripts/ab_prefill.py 2>&1
  B200ATTN_LIB=$L timeout 300 python bench.py --workload prefill --steps 300 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench prefill', round(d['value'],1), d['clocks'])"
  B200ATTN_LIB=$L timeout 300 python bench.py --steps 300 --no-cpu-baseline --no-extra 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench decode', round(d['value'],1), round(d['roofline']['achieved'],1), d['clocks'])"
done
