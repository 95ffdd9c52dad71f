# ncu full capture of the C3-shard slice kernel (1M rows of C2)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_slices" -s 3 -c 1 \
    -o gpurun_out/prof_shard -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 --rows 1000000 > gpurun_out/ncu_shard.log 2>&1
python scripts/ncu_brief.py gpurun_out/prof_shard.ncu-rep > gpurun_out/brief_shard.txt 2>&1
ncu -i gpurun_out/prof_shard.ncu-rep --page source --csv --print-source sass > gpurun_out/shard_sass.csv 2>&1
ls -la gpurun_out/prof_shard.ncu-rep gpurun_out/shard_sass.csv
