# copy-engine block targets (dg_set_block_targets), dg_multi PEER sinks, fused gather modes; C2 unchanged
mkdir -p gpurun_out
timeout 1200 python -m pytest -x -q -m gpu tests/test_fused_gather_gpu.py tests/test_multi_gpu.py tests/test_adapter_gpu.py tests/test_parity_gpu.py 2>&1 | tail -n 3
DG_BENCH_DEVICES=0,0,0,0 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/multi_peer.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/multi_peer.json').read().strip().splitlines()[-1]); print('peer', d['ms_per_step'], d['ms_per_step_kernels'], d['e2e']['ms_per_step'])"
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/p50.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/p50.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['e2e']['ms_per_step'])"
