export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -k "decode or combine or split" > gpurun_out/r2z4_tests.log 2>&1; tail -3 gpurun_out/r2z4_tests.log
LIBAB_OP=decode LIBAB_SHAPES=d1x128,d1x512,d1x2k,d4x512,d16x128 bash scripts/gpujob.sh r2z4 libab > /dev/null 2>&1
python3 - <<'PY'
import json
rows={}
for line in open('gpurun_out/r2z4_libab.log'):
    if line.startswith('{'):
        d=json.loads(line); rows.setdefault(d['shape'],{}).setdefault(d['tag'],[]).append(round(d['us'],2))
for k,v in rows.items(): print(k, v)
PY
