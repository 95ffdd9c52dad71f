# dg_multi: pinned host d downloaded per row block by the shards' doses
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_multi_gpu.py tests/test_adapter_gpu.py tests/test_fused_gather_gpu.py 2>&1 | tail -n 2
for i in 1 2; do
DG_BENCH_DEVICES=0,0,0,0 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/multi_peer.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/multi_peer.json').read().strip().splitlines()[-1]); print('peer x4', d['ms_per_step'], d['ms_per_step_kernels'], d['e2e']['ms_per_step'])"
DG_BENCH_DEVICES=0 timeout 600 python bench.py --engine multi --gather none --steps 20 > gpurun_out/multi_one.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/multi_one.json').read().strip().splitlines()[-1]); print('multi x1', d['ms_per_step'], d['ms_per_step_kernels'], d['e2e']['ms_per_step'])"
done
