# Round-end evidence part 2: sanitizers over the final code, dg_multi on a virtual device list
mkdir -p gpurun_out
SAN_TIMEOUT=700 bash scripts/sanitize.sh
DG_BENCH_DEVICES=0,0,0,0 timeout 600 python bench.py --engine multi --gather peer --steps 20 > gpurun_out/multi_peer.json 2>&1; tail -c 1500 gpurun_out/multi_peer.json
