# Round-end evidence: tests, smoke, bench lines (C2 default + C1/C4/C5 + shard), virtual C3
# shards, the ncu launch list and full captures.  Everything under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.txt 2>&1; tail -n 2 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -n 1 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_c2_30.json 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 20 > gpurun_out/bench_c4.json 2>&1
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/bench_c5.json 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 --rows 1000000 > gpurun_out/bench_shard8.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1
timeout 900 python scripts/virtual_shards.py > gpurun_out/virtual_shards.jsonl 2>&1
timeout 1200 bash scripts/profile_round.sh
# summaries on the box (the .ncu-rep files are too large to bring back: gpurun_out <= 64 MiB)
mkdir -p gpurun_out/prof_summ
cp profiles/dram_bytes_per_launch.json gpurun_out/prof_summ/ 2>/dev/null
DG_PROFILES_OUT=gpurun_out/prof_summ python scripts/summarize_profiles.py r01 > gpurun_out/prof_summ/summarize.log 2>&1
python scripts/ncu_sass_hot.py gpurun_out/prof_exact.ncu-rep dump > gpurun_out/prof_summ/exact_sass_dump.txt 2>&1
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out gpurun_out/prof_summ
