#!/usr/bin/env bash
# One parameterised gpurun job runner (replaces round 1's one-shot scripts/jobs/gpu_r1s*.sh).
#   gpurun --timeout T -- 'bash scripts/gpujob.sh TAG recipe [recipe ...]'
# Each recipe writes gpurun_out/TAG_<recipe>.* ; every step has its own timeout so a hang is cut
# short before gpurun's limit.  Recipes:
#   tests      pytest -m gpu (+ per-config parity table)       smoke     __graft_entry__.smoke()
#   bench      default bench line                               benchref  bench.py --impl reference
#   benchpf    bench.py --workload prefill                      c4        bench.py --workload c4 (full C4 on 1 GPU)
#   dist2      2 ranks on one GPU (gloo) through bench.py's N>1 path, with the gather + oracle check
#   launches   ncu launch lists (gpu__time_duration) of the decode and prefill bench workloads
#   ncupf      ncu --set full of K1 on C3                       ncudec    ncu --set full of K2' on C2
#   sanitize   compute-sanitizer memcheck/racecheck/synccheck on small cases of every kernel
#   sota       scripts/sota.py (same-box library comparators)   single    single-launch vs amortised
#   sotagrid   scripts/sota.py --grid (C5 grid, relative_cdf vs the best library per shape)
#   perf       scripts/perf.py time over the BASELINE shapes
#   mergeab    K2' fused merge vs K3' (plain / PDL behind a late trigger) on the decode shapes
#   flatsweep  K2' CTA count (min tiles per CTA) x fused/K3' merge on small decode shapes
#   pdlab      PDL on/off on latency-bound shapes      dtrace  K2' per-CTA timelines (trace library)
#   narrow     K2' vs K2 on kv-head shards (Hkv = 1/2/4) and batch 4096     e2e   perf.py e2e breakdown
#   libab      two library builds A/B on one box      ptrace  K1 per-CTA launch timelines + C1 trace (trace build)
#   umma       tcgen05 MMA issue-rate probe            c5      the C5 sweep (unmodified ktune tune, exhaustive)
#   pairtests / pairab   CTA-pair K1 parity / A/B      bandtests / bandab   banded K1 order parity / A/B
#   smalldec / mergesmall   small decode shapes (dispatch vs K2', per-CTA timelines), merge modes
#   e2eab      perf.py e2e with two builds (base/new)   pdlcombine  K3' PDL behind a late K2' trigger, on/off
#   smalltime  latency-bound decode shapes: dispatch vs K2' forced      decodetests  the decode/step GPU tests
#   (decode library A/B: LIBAB_OP=decode LIBAB_SHAPES=d1x8k,C2,... with the libab recipe; K2' timelines: dtrace)
set -u
TAG=$1; shift
mkdir -p gpurun_out
export PYTHONPATH=$PWD
O=gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > ${O}_smi.txt 2>&1
for r in "$@"; do
  echo "== $r" >&2
  case $r in
    tests) timeout 1500 python -m pytest tests -m gpu -q -rs > ${O}_tests.log 2>&1; tail -40 ${O}_tests.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; tail -3 ${O}_smoke.log ;;
    bench) timeout 900 python bench.py --steps 20 --warmup 5 > ${O}_bench.json 2> ${O}_bench.err; cat ${O}_bench.json; tail -5 ${O}_bench.err ;;
    benchref) timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > ${O}_benchref.json 2>&1; cat ${O}_benchref.json ;;
    benchpf) timeout 900 python bench.py --workload prefill --steps 50 --warmup 5 --no-cpu-baseline > ${O}_benchpf.json 2>&1; cat ${O}_benchpf.json ;;
    c4) timeout 1200 python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > ${O}_c4.json 2>&1; cat ${O}_c4.json ;;
    dist2) B200_BENCH_ALLOW_SHARED_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
             --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline \
             --dist-backend gloo > ${O}_dist2.json 2> ${O}_dist2.err; cat ${O}_dist2.json; tail -20 ${O}_dist2.err ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches_decode.csv \
        python bench.py --steps 3 --warmup 3 --no-extra --no-cpu-baseline > /dev/null 2>&1
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches_prefill.csv \
        python bench.py --workload prefill --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 ;;
    ncupf) timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_fwd -s 2 -c 1 \
             -o ${O}_pf python scripts/perf.py prof --op prefill > ${O}_ncupf.log 2>&1; tail -3 ${O}_ncupf.log
           # summarised on the box (a full report can push gpurun_out past its copy-back limit)
           python scripts/ncu_summarize.py full ${O}_pf.ncu-rep prefill_fwd_kernel 1291603001344 flops > ${O}_ncupf_summary.txt 2>&1
           ncu -i ${O}_pf.ncu-rep --page raw --csv > ${O}_ncupf_raw.csv 2>/dev/null
           [ -n "${NCU_DROP_REP:-}" ] && rm -f ${O}_pf.ncu-rep ;;
    ncudec) timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_flat -s 2 -c 1 \
             -o ${O}_dec python scripts/perf.py prof --op decode > ${O}_ncudec.log 2>&1; tail -3 ${O}_ncudec.log
           python scripts/ncu_summarize.py full ${O}_dec.ncu-rep decode_flat_kernel 1074856192 bytes > ${O}_ncudec_summary.txt 2>&1
           ncu -i ${O}_dec.ncu-rep --page raw --csv > ${O}_ncudec_raw.csv 2>/dev/null
           [ -n "${NCU_DROP_REP:-}" ] && rm -f ${O}_dec.ncu-rep ;;
    sanitize) timeout 2400 bash scripts/sanitize.sh ${O}_sanitize ;;
    sota) timeout 2400 python scripts/sota.py --out ${O}_sota.json > ${O}_sota.log 2>&1; tail -30 ${O}_sota.log ;;
    sotagrid) timeout 2400 python scripts/sota.py --grid --out ${O}_sotagrid.json > ${O}_sotagrid.log 2>&1; tail -3 ${O}_sotagrid.log ;;
    single) timeout 600 python scripts/perf.py single --shapes C3,C1 > ${O}_single.log 2>&1; cat ${O}_single.log ;;
    perf) timeout 900 python scripts/perf.py time --shapes C1,C3,1x16k,C2,C4shard,C2fp8 > ${O}_perf.log 2>&1; cat ${O}_perf.log ;;
    narrow) for c in '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}' '{"TILE_N": 128, "num_splits": 0, "num_stages": 4}'; do
              timeout 900 python scripts/perf.py time --shapes C2kv2,C2kv1,C4kv1,C4kv4,b4096 --cfg "$c" --tag narrow
            done > ${O}_narrow.log 2>&1; cat ${O}_narrow.log ;;
    pdlab) for v in 1 0; do B200ATTN_PDL=$v timeout 600 python scripts/perf.py time --tag pdl$v \
             --shapes C1,d1x512,d1x8k,d4x2k,d16x512,d64x512,C2; done > ${O}_pdlab.log 2>&1; cat ${O}_pdlab.log ;;
    dtrace) B200ATTN_LIB=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so timeout 600 python scripts/perf.py \
             dtrace --shapes d64x512,d16x512,d1x8k,C2,C4kv1,C2kv2 > ${O}_dtrace.log 2>&1; cat ${O}_dtrace.log ;;
    flatsweep) for mt in 2 4 8 16; do for fm in auto 0; do
               env B200ATTN_FLAT_MIN_TILES=$mt $( [ $fm = 0 ] && echo B200ATTN_FLAT_MERGE=0 ) timeout 300 python scripts/perf.py time \
                 --tag "mt$mt-merge$fm" --shapes d1x512,d1x8k,d4x2k,d16x512,d64x512,C2kv2,C2kv1 \
                 --cfg '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'; done; done > ${O}_flatsweep.log 2>&1
               cat ${O}_flatsweep.log ;;
    mergeab) for v in "" "B200ATTN_FLAT_MERGE=0" "B200ATTN_FLAT_MERGE=0 B200ATTN_PDL_COMBINE=1" "B200ATTN_PDL_COMBINE=1" \
                 "B200ATTN_FLAT_MERGE=0 B200ATTN_PDL_COMBINE=1 B200ATTN_FLAT_MIN_TILES=4"; do
               env $v timeout 300 python scripts/perf.py time --tag "[$v]" --shapes C2,C4shard,C2fp8,d64x512,d1x8k,d16x512,C2kv2,C4kv1
             done > ${O}_mergeab.log 2>&1; cat ${O}_mergeab.log ;;
    e2e) timeout 600 python scripts/perf.py e2e > ${O}_e2e.log 2>&1; cat ${O}_e2e.log ;;
    pfe2e) timeout 900 python scripts/perf.py pfe2e > ${O}_pfe2e.log 2>&1; cat ${O}_pfe2e.log ;;
    bandab) for b in 0 16 8 32; do B200ATTN_PREFILL_BAND=$b timeout 600 python scripts/perf.py time --op prefill \
              --shapes C3,1x16k,4x8k,16x8k,1x32k,16x2k --tag band$b; done > ${O}_bandab.log 2>&1; cat ${O}_bandab.log ;;
    bandtests) timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "banded or c3_full or every_compiled" \
             > ${O}_bandtests.log 2>&1; tail -15 ${O}_bandtests.log ;;
    smalldec) for c in "" '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'; do
              timeout 300 python scripts/perf.py time --op decode --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x512,d16x2k,d64x512,C2 \
                ${c:+--cfg "$c"} --tag "cfg=${c:-dispatch}"; done > ${O}_smalldec.log 2>&1
            B200ATTN_LIB=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so timeout 300 python scripts/perf.py dtrace \
              --shapes d16x512,d4x2k,d1x8k,d64x512 --cfg '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}' >> ${O}_smalldec.log 2>&1
            cat ${O}_smalldec.log ;;
    mergesmall) S=d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x512,d64x512,C2; C='{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'
            { timeout 300 python scripts/perf.py time --op decode --shapes $S --cfg "$C" --partial --tag K2only
              for v in "B200ATTN_FLAT_MERGE=0" "B200ATTN_FLAT_MERGE=1" "B200ATTN_FLAT_MERGE=0 B200ATTN_PDL_COMBINE=1" "B200ATTN_PDL=0"; do
                env $v timeout 300 python scripts/perf.py time --op decode --shapes $S --cfg "$C" --tag "$v"; done; } > ${O}_mergesmall.log 2>&1
            cat ${O}_mergesmall.log ;;
    libab) # two builds on one box, alternating (base = _lib/libb200attn_base.so): LIBAB_OP / LIBAB_SHAPES
            for r in 1 2; do for lib in base new; do
              f=$PWD/paper_2505_03780_b200/_lib/libb200attn.so; [ $lib = base ] && f=$PWD/paper_2505_03780_b200/_lib/libb200attn_base.so
              B200ATTN_LIB=$f timeout 600 python scripts/perf.py time --op ${LIBAB_OP:-prefill} \
                --shapes ${LIBAB_SHAPES:-C1,C3,1x16k,16x2k,16x8k} --tag $lib
            done; done > ${O}_libab.log 2>&1; cat ${O}_libab.log ;;
    ptrace) T=$PWD/paper_2505_03780_b200/_lib/libb200attn_trace.so  # K1 per-CTA launch timelines (trace build)
            for pdl in 1 0; do B200ATTN_PDL=$pdl B200ATTN_LIB=$T timeout 300 python scripts/perf.py ptrace \
              --shapes C1,C3,1x16k --tag "pdl$pdl"; done > ${O}_ptrace.log 2>&1
            B200ATTN_PDL=0 B200ATTN_LIB=$T timeout 300 python scripts/perf.py ptrace --shapes C1 --tag pdl0 --per-cta >> ${O}_ptrace.log 2>&1
            B200ATTN_LIB=$T timeout 300 python scripts/perf.py c1trace --tag pdl1 >> ${O}_ptrace.log 2>&1
            cat ${O}_ptrace.log ;;
    umma) timeout 300 python scripts/perf.py umma-rate > ${O}_umma.log 2>&1; cat ${O}_umma.log ;;
    c5) timeout 5400 python scripts/c5_sweep.py run --out ${O}_c5 --batch 4 > ${O}_c5_run.log 2>&1
        rm -rf ${O}_c5/cache; tail -5 ${O}_c5_run.log ;;
    pairtests) timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pair or every_compiled" \
             > ${O}_pairtests.log 2>&1; tail -15 ${O}_pairtests.log ;;
    pairab) for c in '{"BLOCK_M": 256, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1, "PRE_LOAD_V": false}' \
                     '{"BLOCK_M": 256, "BLOCK_N": 128, "num_warps": 4, "num_stages": 1, "waves_per_eu": 2, "PRE_LOAD_V": false}' \
                     '{"BLOCK_M": 256, "BLOCK_N": 128, "num_warps": 4, "num_stages": 2, "waves_per_eu": 2, "PRE_LOAD_V": false}' \
                     '{"BLOCK_M": 256, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 2, "PRE_LOAD_V": false}' \
                     '{"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 4, "num_stages": 2, "waves_per_eu": 2, "PRE_LOAD_V": false}' \
                     '{"BLOCK_M": 128, "BLOCK_N": 128, "num_warps": 4, "num_stages": 3, "waves_per_eu": 1, "PRE_LOAD_V": false}'; do
              timeout 300 python scripts/perf.py time --op prefill --shapes C3,1x16k,4x8k,C1 --cfg "$c" --tag "$c"
            done > ${O}_pairab.log 2>&1; cat ${O}_pairab.log ;;
    e2eab) # DecodeStep e2e breakdown (perf.py e2e) with two library builds alternating (base = _lib/libb200attn_base.so)
            for rr in 1 2; do for lib in base new; do
              f=$PWD/paper_2505_03780_b200/_lib/libb200attn.so; [ $lib = base ] && f=$PWD/paper_2505_03780_b200/_lib/libb200attn_base.so
              B200ATTN_LIB=$f timeout 300 python scripts/perf.py e2e --tag $lib
            done; done > ${O}_e2eab.log 2>&1; cat ${O}_e2eab.log ;;
    pdlcombine) for v in 0 1; do B200ATTN_PDL_COMBINE=$v timeout 300 python scripts/perf.py time --tag pdlc$v \
                  --shapes d1x2k,d1x8k,d4x2k,d16x512,d64x512,C2 --cfg '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}'; done \
                  > ${O}_pdlcombine.log 2>&1; cat ${O}_pdlcombine.log ;;
    smalltime) # the C5 grid's latency-bound decode shapes: shipped dispatch vs K2' forced
            timeout 600 python scripts/perf.py time --tag dispatch \
              --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x128,d16x512,d64x512,C2 > ${O}_smalltime.log 2>&1
            timeout 600 python scripts/perf.py time --tag flat --cfg '{"TILE_N": 16, "num_splits": 0, "num_stages": 4}' \
              --shapes d1x128,d1x512,d1x2k,d1x8k,d4x512,d4x2k,d16x128,d16x512,d64x512,C2 >> ${O}_smalltime.log 2>&1
            cat ${O}_smalltime.log ;;
    decodetests) timeout 900 python -m pytest tests -q -m gpu -k "decode or flat or combine or split or step" \
                   > ${O}_decodetests.log 2>&1; tail -3 ${O}_decodetests.log ;;
    *) echo "unknown recipe $r" >&2 ;;
  esac
done
