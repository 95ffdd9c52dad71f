#!/bin/bash
# One GPU session: parity tests, bench, launch list, one full ncu capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/gpu_tests.txt
python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --accum fp32 --no-cpu-baseline > gpurun_out/bench_fp32.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:warp_exact -s 3 -c 1 \
    -o gpurun_out/prof_warp_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
