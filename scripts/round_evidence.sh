# Round-end evidence: GPU tests, smoke, bench lines (C2 driver-style 20 steps and 100 steps,
# C1/C4/C5, 1/8 shard), reference arm, virtual C3 shards, the ncu launch list and full captures,
# summarised on the box into gpurun_out/prof_summ (the .ncu-rep files stay there).
#   TAG=r02 bash scripts/round_evidence.sh
TAG=${TAG:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.txt 2>&1; tail -n 2 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -n 1 gpurun_out/smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_20.json 2> gpurun_out/bench_c2_20.err
timeout 900 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_c2_100.json 2>&1
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 20 > gpurun_out/bench_c4.json 2>&1
timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 > gpurun_out/bench_c5.json 2>&1
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 --rows 1000000 > gpurun_out/bench_shard8.json 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1
timeout 900 python scripts/virtual_shards.py > gpurun_out/virtual_shards.jsonl 2>&1
timeout 1500 bash scripts/profile_round.sh
mkdir -p gpurun_out/prof_summ
cp profiles/dram_bytes_per_launch.json gpurun_out/prof_summ/ 2>/dev/null
DG_PROFILES_OUT=gpurun_out/prof_summ python scripts/summarize_profiles.py $TAG > gpurun_out/prof_summ/summarize.log 2>&1
for f in exact fp32 c4; do
  python scripts/ncu_brief.py gpurun_out/prof_$f.ncu-rep > gpurun_out/prof_summ/brief_$f.txt 2>&1
done
ls -la gpurun_out gpurun_out/prof_summ
