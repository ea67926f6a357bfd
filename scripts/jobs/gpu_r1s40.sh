set -x
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r1s40_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1s40_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r1s40_bench.json 2> gpurun_out/r1s40_bench.err
cat gpurun_out/r1s40_pytest.log gpurun_out/r1s40_smoke.log gpurun_out/r1s40_bench.json
