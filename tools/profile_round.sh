#!/bin/bash
# One profiling pass on a B200 (run under gpurun from the repo root).
# Outputs under gpurun_out/; summarised into profiles/ by tools/summarize_profiles.py.
set -x
OUT=gpurun_out/prof
mkdir -p $OUT
# 1. the bench line (plain, no profiler)
python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
# 2. launch list of the same command (shortened: shares, not absolutes)
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/plain_short.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
# 3. full captures of the top kernels (1 launch each, after their plain runs exited 0)
python tools/prof_router.py --iters 1 > $OUT/router_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_router -s 2 -c 1 \
    -o $OUT/router_full python tools/prof_router.py --iters 1 > $OUT/ncu_router.log 2>&1
python tools/kbench.py > $OUT/kbench_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_layout_count|k_layout_scatter|k_layout_scan|k_coact_partial|k_score|k_finalize" \
    -s 6 -c 8 -o $OUT/small_full python tools/kbench.py > $OUT/ncu_small.log 2>&1
ls -la $OUT
