export PYTHONPATH=$PWD
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_TRACE -o /tmp/libtrace.so paper_2505_03780_b200/csrc/capi.cu > /dev/null 2>&1
B200ATTN_LIB=/tmp/libtrace.so timeout 300 python scripts/trace_prefill.py 2>&1 | head -16
