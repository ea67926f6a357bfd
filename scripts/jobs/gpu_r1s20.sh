export PYTHONPATH=$PWD
timeout 1500 python scripts/c5_sweep.py run --extra-only --out gpurun_out/c5x > gpurun_out/c5x_run.log 2>&1
rm -rf gpurun_out/c5x/cache
cat gpurun_out/c5x_run.log
