export PYTHONPATH=$PWD
L=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so
B200ATTN_PDL=0 B200ATTN_LIB=$L timeout 300 python scripts/perf.py ptrace --shapes C1 --tag pdl0 --per-cta > gpurun_out/${1}_ptrace2.log 2>&1
