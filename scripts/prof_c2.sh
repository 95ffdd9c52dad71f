# step overhead + bench + full ncu capture of the C2 exact tile kernel (source counters)
mkdir -p gpurun_out
timeout 300 python scripts/step_overhead.py > gpurun_out/step_overhead.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 3 -c 1 \
    -o gpurun_out/prof_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/ncu_exact.log 2>&1
cat gpurun_out/step_overhead.txt gpurun_out/bench_c2.json; tail -2 gpurun_out/ncu_exact.log
