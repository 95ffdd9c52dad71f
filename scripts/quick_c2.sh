#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_scatter_gpu.py -x -q -s -m gpu -k gather 2>&1 | tail -4 > gpurun_out/gpu_scatter.txt
python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_c2.json 2>gpurun_out/bench.err
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_tiles -s 2 -c 1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/ncu_dram.txt 2>&1
