# final-tree confirmation: GPU tests + smoke + default bench
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r1s59_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s59_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s59_bench.json 2> gpurun_out/r1s59_bench.err
cat gpurun_out/r1s59_pytest.log gpurun_out/r1s59_smoke.log
python -c "import json; d=json.loads(open('gpurun_out/r1s59_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['extra']['prefill_C3']['TFLOP/s'])"
