#!/bin/bash
# Round evidence: launch list of the bench command + one full ncu capture of the hot kernel
# (exact and fp32 families).  Summaries are copied into profiles/ by scripts/summarize_profiles.py.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(slices|tiles|dense)" -s 2 -c 2 \
    -o gpurun_out/prof_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(slices|tiles|dense)" -s 2 -c 2 \
    -o gpurun_out/prof_fp32 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --accum fp32 > gpurun_out/ncu_fp32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(slices|tiles)" -s 1 -c 1 \
    -o gpurun_out/prof_c4 -f python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/ncu_c4.log 2>&1
tail -n 2 gpurun_out/ncu_exact.log gpurun_out/ncu_fp32.log gpurun_out/ncu_c4.log
