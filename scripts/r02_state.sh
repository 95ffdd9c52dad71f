# r02 state check: ncu full of the C2 dose kernels (exact + fp32), launch list, C4 / C3-shard / C1 bench lines
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/r02_launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(slices|dense)" -s 2 -c 2 \
    -o gpurun_out/r02_exact -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 > gpurun_out/r02_ncu_exact.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_(slices|dense)" -s 2 -c 2 \
    -o gpurun_out/r02_fp32 -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --accum fp32 --no-alt-fp32 > gpurun_out/r02_ncu_fp32.log 2>&1
for r in exact fp32; do python scripts/ncu_brief.py gpurun_out/r02_$r.ncu-rep > gpurun_out/r02_brief_$r.txt 2>&1; done
timeout 600 python bench.py --config c4 --no-cpu-baseline --no-alt-fp32 --steps 20 > gpurun_out/r02_c4.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 30 --rows 1000000 > gpurun_out/r02_shard8.json 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline --no-alt-fp32 > gpurun_out/r02_c1.json 2>&1
tail -c 1500 gpurun_out/r02_c4.json; tail -c 600 gpurun_out/r02_shard8.json; tail -c 600 gpurun_out/r02_c1.json
cat gpurun_out/r02_brief_exact.txt
ls -la gpurun_out
