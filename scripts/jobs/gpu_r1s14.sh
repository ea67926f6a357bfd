export PYTHONPATH=$PWD
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --use_fast_math -Xcompiler -fPIC -shared -Iinclude -DB200_TRACE -o /tmp/libtrace.so paper_2505_03780_b200/csrc/capi.cu > /dev/null 2>&1
B200ATTN_LIB=/tmp/libtrace.so timeout 300 python scripts/trace_prefill.py 2>&1 | head -24
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jumps" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 -o gpurun_out/pf_r1s14 python scripts/prof_target.py prefill > /dev/null 2>&1
ls gpurun_out/pf_r1s14*
