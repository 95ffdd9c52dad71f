# compute-sanitizer over the sanitize_run.py workload, one tool at a time -> gpurun_out/sanitizer_<tool>.txt
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck racecheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  [ "$tool" = "initcheck" ] && extra=""
  q=""; [ "$tool" = "racecheck" ] && q="--quick"
  timeout ${SAN_TIMEOUT:-800} compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
      python scripts/sanitize_run.py $q > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
  tail -n 4 gpurun_out/sanitizer_$tool.txt
done
