# A/B: producer-side nanosleep backoff (B200_PRODUCER_SLEEP_NS) on prefill; traces of both
mkdir -p gpurun_out
export PYTHONPATH=$PWD
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude"



for rep in 1 2; do
timeout 300 python scripts/ab_prefill.py 2>&1 | sed "s/^/base /"
for ns in 20 100; do B200ATTN_LIB=_ab/lib_sleep$ns.so timeout 300 python scripts/ab_prefill.py 2>&1 | sed "s/^/sleep$ns /"; done
done > gpurun_out/r1s47_ab.txt
for v in 0 20; do B200ATTN_LIB=_ab/libtrace$v.so timeout 300 python scripts/trace_prefill.py 256 2 4 2>&1 | tail -6 | sed "s/^/trace$v /"; done >> gpurun_out/r1s47_ab.txt
cat gpurun_out/r1s47_ab.txt
