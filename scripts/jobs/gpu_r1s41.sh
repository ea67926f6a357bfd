mkdir -p gpurun_out
export PYTHONPATH=$PWD
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_probe scripts/probes/mufu_probe.cu && /tmp/mufu_probe > gpurun_out/r1s41_mufu.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_TRACE -o /tmp/libtrace.so paper_2505_03780_b200/csrc/capi.cu > gpurun_out/r1s41_tracebuild.log 2>&1
B200ATTN_LIB=/tmp/libtrace.so timeout 300 python scripts/trace_prefill.py > gpurun_out/r1s41_trace.txt 2>&1
cat gpurun_out/r1s41_mufu.txt; head -30 gpurun_out/r1s41_trace.txt
