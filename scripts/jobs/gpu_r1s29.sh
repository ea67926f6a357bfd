export PYTHONPATH=$PWD
timeout 900 python scripts/c5_sweep.py run --ops prefill --batch 8 --cooldown-ms 500 --shapes scripts/jobs/c3_shape.json --out gpurun_out/c5g > gpurun_out/c5g_run.log 2>&1
rm -rf gpurun_out/c5g/cache; tail -1 gpurun_out/c5g_run.log
