export PYTHONPATH=$PWD
timeout 1700 python scripts/c5_sweep.py run --ops prefill --batch 4 --shapes scripts/jobs/c5d_missing_shapes.json --out gpurun_out/c5e > gpurun_out/c5e_run.log 2>&1
rm -rf gpurun_out/c5e/cache
tail -2 gpurun_out/c5e_run.log
