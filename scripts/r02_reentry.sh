# Re-entry check on HEAD: GPU suite, smoke, C2 headline (driver-style), C3 shard
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.txt 2>&1; tail -n 3 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -n 2 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_20.json 2> gpurun_out/bench_c2_20.err; tail -c 600 gpurun_out/bench_c2_20.json
timeout 300 python bench.py --no-cpu-baseline --steps 30 --rows 1000000 > gpurun_out/bench_shard8.json 2>&1; tail -c 300 gpurun_out/bench_shard8.json
