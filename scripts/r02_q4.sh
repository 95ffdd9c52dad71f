set -x
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print(d['ms_per_step'],d['roofline']['kernels'],d['e2e']['ms_per_step'],d['alt_fp32']['ms_per_step'])"
for rw in 1 2 3; do DG_RUNS_PER_WARP=$rw timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-alt-fp32 > gpurun_out/q_rw$rw.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/q_rw$rw.json'));print('rw $rw', d['ms_per_step'],d['roofline']['kernels'])"; done
for rw in 1 2 3; do DG_RUNS_PER_WARP=$rw timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-alt-fp32 --rows 1000000 > gpurun_out/q_s8rw$rw.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/q_s8rw$rw.json'));print('shard rw $rw', d['ms_per_step'],d['roofline']['kernels'])"; done
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py 2>&1 | grep -v "^ " | head -6
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py --rows 1000000 2>&1 | grep -v "^ " | head -6
