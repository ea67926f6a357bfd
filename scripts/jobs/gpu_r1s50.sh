# A/B: share of exponentials on the FMA pipe (B200_PREFILL_EMU) with the setmaxnreg prefill kernel
mkdir -p gpurun_out
export PYTHONPATH=$PWD
for rep in 1 2; do
timeout 300 python scripts/ab_prefill.py 2>&1 | sed "s/^/emu3 /"
for e in 0 2 4 6; do B200ATTN_LIB=_ab/lib_emu$e.so timeout 300 python scripts/ab_prefill.py 2>&1 | sed "s/^/emu$e /"; done
done > gpurun_out/r1s50_ab.txt
cat gpurun_out/r1s50_ab.txt
