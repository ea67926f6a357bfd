# EARLY S release (prefill): parity, A/B against EARLY=0, trace
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" 2>&1 | tail -5 > gpurun_out/r1s51_pytest.log
cat gpurun_out/r1s51_pytest.log
for rep in 1 2; do
timeout 200 python scripts/ab_prefill.py 2>&1 | sed "s/^/early1 /"
B200ATTN_LIB=_ab/lib_early0.so timeout 200 python scripts/ab_prefill.py 2>&1 | sed "s/^/early0 /"
done > gpurun_out/r1s51_ab.txt
B200ATTN_LIB=_ab/libtrace_early.so timeout 200 python scripts/trace_prefill.py 256 2 4 2>&1 | tail -8 >> gpurun_out/r1s51_ab.txt
cat gpurun_out/r1s51_ab.txt
