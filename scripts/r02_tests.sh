# full GPU suite + the C2 headline at 20 and 100 steps
set -x
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/t_bench100.json 2>&1; tail -c 1500 gpurun_out/t_bench100.json
