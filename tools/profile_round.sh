#!/bin/bash
# One profiling pass on a B200 (run under gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/profile_round.sh'
# Outputs under gpurun_out/prof/; summarised into profiles/ by
#   python tools/summarize_profiles.py r02
# Every ncu command runs only after the same command exited 0 without ncu.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
# ncu reports are exported to CSV on the box and removed (gpurun copies back <= 64 MiB)
export_rep() {
  ncu -i $1.ncu-rep --page raw --csv > $1.raw.csv 2>/dev/null
  ncu -i $1.ncu-rep --page details --csv > $1.details.csv 2>/dev/null
  ncu -i $1.ncu-rep --page source --csv --print-source sass > $1.source.csv 2>/dev/null
  gzip -f $1.source.csv $1.details.csv
  rm -f $1.ncu-rep
}
# 1. plain bench lines (no profiler), one per BASELINE workload
for W in dsv3 qwen3 maverick domain; do
  python bench.py --workload $W > $OUT/bench_$W.json 2> $OUT/bench_$W.err
done
# 2. launch lists of the same commands (shortened: shares, not absolutes)
for W in dsv3 qwen3; do
  CMD="python bench.py --workload $W --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-a2a"
  $CMD > $OUT/plain_$W.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$W.csv $CMD > $OUT/ncu_launches_$W.log 2>&1
done
# 3. router: full capture of one launch per workload shape (+ cuBLAS timing line)
declare -A SHAPE=( [dsv3]="--T 65536 --H 7168 --E 256 --k 8 --fn 1"
                   [qwen3]="--T 4096 --H 4096 --E 128 --k 8 --fn 0"
                   [maverick]="--T 1048576 --H 5120 --E 128 --k 1 --fn 1"
                   [domain]="--T 1048576 --H 4096 --E 128 --k 8 --fn 0" )
for W in dsv3 qwen3 maverick domain; do
  python tools/prof_router.py ${SHAPE[$W]} --iters 5 > $OUT/router_plain_$W.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_router -s 2 -c 1 \
      -o $OUT/router_$W python tools/prof_router.py ${SHAPE[$W]} --iters 1 > $OUT/ncu_router_$W.log 2>&1
  export_rep $OUT/router_$W
done
python tools/prof_router.py --layers 8 --iters 5 > $OUT/router_grouped_plain.log 2>&1
# 4. statistics / scoring kernels: full captures at the DSv3 step shape (tools/kbench.py),
#    the co-activation tcgen05 kernel and the scorer included
python tools/kbench.py > $OUT/kbench_plain.log 2>&1
python tools/kbench.py --once > $OUT/kbench_once.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_layout_count|k_layout_scan|k_layout_scatter|k_coact_mma|k_score|k_finalize" \
    -c 20 -o $OUT/small_full python tools/kbench.py --once > $OUT/ncu_small.log 2>&1
export_rep $OUT/small_full
gzip -f $OUT/launches_dsv3.csv $OUT/launches_qwen3.csv
ls -la $OUT
