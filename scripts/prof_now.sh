#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 1 -c 1 \
    -o gpurun_out/prof_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/ncu_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 6 -c 2 \
    -o gpurun_out/prof_c4 -f python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_exact.log gpurun_out/ncu_c4.log
