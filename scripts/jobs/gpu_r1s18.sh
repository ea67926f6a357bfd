export PYTHONPATH=$PWD
timeout 3000 python scripts/c5_sweep.py run --ops prefill --out gpurun_out/c5c > gpurun_out/c5c_run.log 2>&1
rm -rf gpurun_out/c5c/cache
tail -2 gpurun_out/c5c_run.log
