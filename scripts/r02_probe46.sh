# rotated value-stream lane grid (DG_VALUES_ROT): parity, then interleaved C2 / C3-shard A/B
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_parity_gpu.py tests/test_fuzz_gpu.py > gpurun_out/p46_tests.txt 2>&1; tail -n 2 gpurun_out/p46_tests.txt
timeout 900 python -m pytest -x -q -m gpu tests/test_fullscale_gpu.py -k "c2_full or pinned or c3_shards" >> gpurun_out/p46_tests.txt 2>&1; tail -n 2 gpurun_out/p46_tests.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -n 2
for i in 1 2 3; do
for r in 0 1; do
  DG_VALUES_ROT=$r timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/p46.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p46.json').read().strip().splitlines()[-1])
print('ROT=$r C2', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()}, d['clocks']['sm_mhz'])"
  DG_VALUES_ROT=$r timeout 300 python bench.py --no-cpu-baseline --steps 30 --rows 1000000 > gpurun_out/p46.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p46.json').read().strip().splitlines()[-1])
print('ROT=$r shard', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})"
done; done
