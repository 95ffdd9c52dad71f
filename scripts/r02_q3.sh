set -x
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py 2>&1 | grep -v "^ " | tail -12
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py --accum fp32 2>&1 | grep -v "^ " | tail -12
timeout 2400 compute-sanitizer --tool racecheck --num-cuda-barriers 8 --racecheck-report hazard --error-exitcode 99 --print-limit 20 python scripts/sanitize_run.py --quick > gpurun_out/sanitizer_racecheck_nb.txt 2>&1; echo rc=$?; tail -3 gpurun_out/sanitizer_racecheck_nb.txt
timeout 2400 compute-sanitizer --tool initcheck --error-exitcode 99 --print-limit 20 python scripts/sanitize_run.py > gpurun_out/sanitizer_initcheck.txt 2>&1; echo rc=$?; tail -3 gpurun_out/sanitizer_initcheck.txt
