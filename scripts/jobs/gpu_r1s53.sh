# C5 prefill re-sweep: the shapes of half B that r1s48 did not reach
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 3000 python scripts/c5_sweep.py run --ops prefill --batch 4 --shapes scripts/jobs/c5h_shapes_b2.json --out gpurun_out/c5h > gpurun_out/c5h_b2_run.log 2>&1
rm -rf gpurun_out/c5h/cache
ls gpurun_out/c5h/prefill_results | wc -l
