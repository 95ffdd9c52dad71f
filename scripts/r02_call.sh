set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
cat gpurun_out/c1_bench.json
ncu --set full --clock-control none --import-source on -k regex:k_tiles -s 3 -c 1 -o gpurun_out/r02_tiles_base -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c1_ncu.log 2>&1
tail -3 gpurun_out/c1_ncu.log
ls -la gpurun_out/
