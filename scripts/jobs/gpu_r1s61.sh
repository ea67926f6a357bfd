# A/B: producer-warpgroup register count (softmax gets the rest): 64 (default) vs 40 / 48 / 96
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for rep in 1 2; do
timeout 200 python scripts/ab_prefill.py 2>&1 | grep -v C1 | sed "s/^/reg64 /"
for r in 40 48 96; do B200ATTN_LIB=_ab/lib_reg$r.so timeout 200 python scripts/ab_prefill.py 2>&1 | grep -v C1 | sed "s/^/reg$r /"; done
done > gpurun_out/r1s61_ab.txt
sort gpurun_out/r1s61_ab.txt
