#!/bin/bash
# Profile one kernel of the C2 bench: scripts/gpu_prof.sh <kernel-regex> <skip> <tag> [bench args...]
K=$1; S=$2; TAG=$3; shift 3
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 \
    -o gpurun_out/prof_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
