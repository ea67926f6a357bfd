# C5 prefill re-sweep (half B + the C3 row) with the num_warps=8 variants
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 2700 python scripts/c5_sweep.py run --ops prefill --batch 4 --shapes scripts/jobs/c5h_shapes_b.json --out gpurun_out/c5h > gpurun_out/c5h_b_run.log 2>&1
timeout 600 python scripts/c5_sweep.py run --ops prefill --batch 8 --cooldown-ms 500 --shapes scripts/jobs/c3_shape.json --out gpurun_out/c5h > gpurun_out/c5h_c3_run.log 2>&1
rm -rf gpurun_out/c5h/cache
tail -3 gpurun_out/c5h_b_run.log gpurun_out/c5h_c3_run.log; ls gpurun_out/c5h/prefill_results | wc -l
