# A/B of two builds of the library on the same box: perf.py time with B200ATTN_LIB alternating
#   bash scripts/jobs/libab.sh TAG OP SHAPES   (base = _lib/libb200attn_base.so, new = _lib/libb200attn.so)
export PYTHONPATH=$PWD
O=gpurun_out/${1}; OP=${2:-prefill}; S=${3:-C1,C3,1x16k,16x2k,16x8k}
for r in 1 2; do for lib in base new; do
  f=$PWD/paper_2505_03780_b200/_lib/libb200attn.so; [ $lib = base ] && f=$PWD/paper_2505_03780_b200/_lib/libb200attn_base.so
  B200ATTN_LIB=$f timeout 600 python scripts/perf.py time --op $OP --shapes $S --tag $lib
done; done > ${O}_libab.log 2>&1
