#!/bin/bash
# compute-sanitizer over every kernel family at small shapes (run on a B200
# under gpurun from the repo root). Logs -> gpurun_out/sanitize/, summarised
# into profiles/r02_sanitize.txt.
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for part in router layout coact score kmeans a2a; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 $CS --tool $tool --target-processes all --print-limit 20 \
        python tools/sanitize_driver.py $part > $OUT/${part}_${tool}.log 2>&1
    echo "$part $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/${part}_${tool}.log | tail -1)"
  done
done | tee $OUT/summary.txt
