# dg_multi PEER gather with block-overlapped copies: tests, then the multi bench (virtual device list)
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_multi_gpu.py tests/test_adapter_gpu.py 2>&1 | tail -n 3
for i in 1 2; do
DG_BENCH_DEVICES=0,0,0,0 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/p49.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/p49.json').read().strip().splitlines()[-1]); print('peer', d['ms_per_step'], d['ms_per_step_kernels'], d['e2e']['ms_per_step'])"
DG_BENCH_DEVICES=0,0,0,0 DG_NO_OVERLAP=1 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/p49b.json 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/p49b.json').read().strip().splitlines()[-1]); print('peer no-overlap', d['ms_per_step'], d['ms_per_step_kernels'], d['e2e']['ms_per_step'])"
done
cp gpurun_out/p49.json gpurun_out/multi_peer.json
