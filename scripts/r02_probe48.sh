# tile kernel with two batches in flight per warp (DG_TILE_CFG 40/41/42 = 24/28/20 warps) vs default
mkdir -p gpurun_out
DG_TILE_CFG=40 timeout 900 python -m pytest -x -q -m gpu tests/test_parity_gpu.py tests/test_fuzz_gpu.py 2>&1 | tail -n 2
for i in 1 2; do
for c in 0 40 41 42; do
  DG_TILE_CFG=$c timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 20 --warmup 5 > gpurun_out/p48.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p48.json').read().strip().splitlines()[-1])
print('cfg=$c C2', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()}, d['clocks']['sm_mhz'])"
done
for c in 0 40; do
  DG_TILE_CFG=$c timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 30 --rows 1000000 > gpurun_out/p48.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p48.json').read().strip().splitlines()[-1])
print('cfg=$c shard', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})"
done; done
