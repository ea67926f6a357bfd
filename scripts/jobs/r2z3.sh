export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "decode or flat or combine or step" > gpurun_out/r2z3_tests.log 2>&1; tail -3 gpurun_out/r2z3_tests.log
LIBAB_OP=decode LIBAB_SHAPES=d1x2k,d1x8k,d4x2k,d16x512,d64x512,C2,C4shard,C2fp8,b1x32k,C2kv2 bash scripts/gpujob.sh r2z3 libab > /dev/null 2>&1
cat gpurun_out/r2z3_libab.log
