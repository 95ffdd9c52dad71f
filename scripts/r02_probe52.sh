# value kernel with an x prefetched into L1 one batch ahead (DG_VALUES_CFG 4)
mkdir -p gpurun_out
DG_VALUES_CFG=4 timeout 600 python -m pytest -x -q -m gpu tests/test_parity_gpu.py -k "contiguous" 2>&1 | tail -n 1
for i in 1 2; do
for c in 0 4; do
  DG_VALUES_CFG=$c timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 30 --rows 1000000 > gpurun_out/p51.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p51.json').read().strip().splitlines()[-1])
print('cfg=$c shard', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})"
  DG_VALUES_CFG=$c timeout 300 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 20 --warmup 5 > gpurun_out/p51.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p51.json').read().strip().splitlines()[-1])
print('cfg=$c C2', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()}, d['clocks']['sm_mhz'])"
done; done
