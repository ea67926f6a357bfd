export PYTHONPATH=$PWD
timeout 3000 python scripts/c5_sweep.py run --ops prefill --batch 4 --out gpurun_out/c5d > gpurun_out/c5d_run.log 2>&1
rm -rf gpurun_out/c5d/cache
tail -2 gpurun_out/c5d_run.log
