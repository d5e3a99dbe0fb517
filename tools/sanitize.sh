#!/usr/bin/env bash
# compute-sanitizer over every kernel family (small workloads, tools/sanitize_cases.py):
# memcheck (+ leak check), racecheck (shared-memory hazards), synccheck (barrier misuse),
# initcheck (reads of uninitialised device memory).  Summaries -> gpurun_out/sanitize_*.log
mkdir -p gpurun_out
cases="${CASES:-k2 k3 tick mlp ingest metrics}"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $cases; do
    extra=""
    [ "$tool" = memcheck ] && extra="--leak-check full"
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_${tool}_${c}.log | tr '\n' ' ')"
  done
done | tee gpurun_out/sanitize_summary.txt
