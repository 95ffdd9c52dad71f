# values-after host path: parity (contiguous-row test, C2 pinned path with alternating x), then
# interleaved C2 end-to-end A/B (DG_VALUES_AFTER=0 is the previous values-first order)
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_parity_gpu.py -k "contiguous_rows" > gpurun_out/p41_tests.txt 2>&1; tail -n 3 gpurun_out/p41_tests.txt
timeout 900 python -m pytest -x -q -m gpu tests/test_fullscale_gpu.py -k "pinned_host" >> gpurun_out/p41_tests.txt 2>&1; tail -n 3 gpurun_out/p41_tests.txt
for i in 1 2; do
for va in 0 1; do
  DG_VALUES_AFTER=$va timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/p41_va$va.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p41_va$va.json').read().strip().splitlines()[-1])
print('VA=$va', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
for va in 0 1; do DG_VALUES_AFTER=$va timeout 300 python scripts/e2e_probe.py; done
