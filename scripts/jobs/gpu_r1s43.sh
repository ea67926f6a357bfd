mkdir -p gpurun_out
export PYTHONPATH=$PWD
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_TRACE -o /tmp/libtrace.so paper_2505_03780_b200/csrc/capi.cu > gpurun_out/r1s43_tracebuild.log 2>&1
for c in "256 1 4" "256 1 8" "256 2 8"; do
B200ATTN_LIB=/tmp/libtrace.so timeout 300 python scripts/trace_prefill.py $c 2>&1 | tail -12
done > gpurun_out/r1s43_trace.txt
cat gpurun_out/r1s43_trace.txt
