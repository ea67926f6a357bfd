# bench (packed e2e copies) + C5 prefill re-sweep (half A) with the num_warps=8 variants
mkdir -p gpurun_out
export PYTHONPATH=$PWD
timeout 600 python bench.py > gpurun_out/r1s46_bench.json 2> gpurun_out/r1s46_bench.err
timeout 2400 python scripts/c5_sweep.py run --ops prefill --batch 4 --shapes scripts/jobs/c5h_shapes_a.json --out gpurun_out/c5h > gpurun_out/c5h_a_run.log 2>&1
rm -rf gpurun_out/c5h/cache
cat gpurun_out/r1s46_bench.json; tail -3 gpurun_out/c5h_a_run.log; ls gpurun_out/c5h/prefill_results | wc -l
