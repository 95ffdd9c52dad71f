# bench: C4 optimisation-loop x_k; bench contract tests
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_bench_gpu.py 2>&1 | tail -n 2
timeout 600 python bench.py --config c4 --no-cpu-baseline --steps 20 > gpurun_out/p47_c4.json 2>&1; tail -c 1200 gpurun_out/p47_c4.json
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/p47_c2.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/p47_c2.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['x'])"
