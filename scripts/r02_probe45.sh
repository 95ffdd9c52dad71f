# value-stream share rule: GPU suite, smoke, C1 / C2 / C4 benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.txt 2>&1; tail -n 3 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -n 2
for c in c1 c2 c4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/p45_$c.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p45_$c.json').read().strip().splitlines()[-1])
print('$c', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})"
done
