# r02 baseline on the GPU: full GPU test suite, then the C2 headline bench (driver-style and 100 steps)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench20.json 2> gpurun_out/r02_bench20.err; cat gpurun_out/r02_bench20.json
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench100.json 2>&1; cat gpurun_out/r02_bench100.json | tail -c 3000
