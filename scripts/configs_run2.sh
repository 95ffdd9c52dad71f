#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.txt
python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>>gpurun_out/bench.err
python bench.py --config c4 --no-cpu-baseline --steps 10 > gpurun_out/bench_c4.json 2>>gpurun_out/bench.err
python bench.py --config c5 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_c5.json 2>>gpurun_out/bench.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/bench.err
