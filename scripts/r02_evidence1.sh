set -x
nproc; free -g | head -2
timeout 2400 python -m pytest tests/test_fullscale_gpu.py -x -q -s -k "full_vector" 2>&1 | tail -8
bash scripts/sanitize.sh
DG_BENCH_DEVICES=0,0,0,0 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/multi_peer.json 2>&1; tail -c 1200 gpurun_out/multi_peer.json
timeout 600 python bench.py --engine multi --gpus 1 --gather nccl --steps 20 > gpurun_out/multi_nccl.json 2>&1; tail -c 600 gpurun_out/multi_nccl.json
