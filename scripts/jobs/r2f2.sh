# final evidence, part 2: ingest PDL trigger A/B (perf.py e2e, base = no trigger), e2e bench line,
# sanitizers, same-box SOTA (BASELINE shapes + C5 grid), ncu full capture of K1 on C3
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for r in 1 2; do for lib in base new; do
  f=$PWD/paper_2505_03780_b200/_lib/libb200attn.so; [ $lib = base ] && f=$PWD/paper_2505_03780_b200/_lib/libb200attn_base.so
  B200ATTN_LIB=$f timeout 300 python scripts/perf.py e2e --tag $lib
done; done > gpurun_out/r2f2_e2eab.log 2>&1; cat gpurun_out/r2f2_e2eab.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f2_bench.json 2> gpurun_out/r2f2_bench.err; tail -c 600 gpurun_out/r2f2_bench.json
NCU_DROP_REP=1 bash scripts/gpujob.sh r2f2 sanitize sotagrid sota ncupf
