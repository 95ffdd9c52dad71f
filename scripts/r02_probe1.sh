# per-warp streaming rate microbenchmark, shard tile timeline, racecheck after the all-lane arrive
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -diag-suppress 186 -o /tmp/stream_rate scripts/micro/stream_rate.cu && timeout 300 /tmp/stream_rate > gpurun_out/stream_rate.txt 2>&1
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py --rows 1000000 > gpurun_out/trace_shard.txt 2>&1
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py > gpurun_out/trace_c2.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 20 > gpurun_out/p1_c2.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 30 --rows 1000000 > gpurun_out/p1_shard8.json 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 99 --print-limit 20 python scripts/sanitize_run.py --quick > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?"
tail -3 gpurun_out/sanitizer_racecheck.txt
cat gpurun_out/stream_rate.txt
