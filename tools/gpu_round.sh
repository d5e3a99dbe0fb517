mkdir -p gpurun_out
for tool in racecheck synccheck memcheck; do
  extra=""; [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py tick_full > gpurun_out/sanitize_${tool}_tick_full.log 2>&1
  echo "$tool tick_full rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_${tool}_tick_full.log | tr '\n' ' ')"
done > gpurun_out/r2s3_sanitize_tickfull.txt
