#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/gpu_tests.txt
for c in 0 1 2 3 4; do
  DG_TILE_CFG=$c python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg$c.json 2>>gpurun_out/bench.err
done
DG_TILE_NNZ=131072 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_t128k.json 2>>gpurun_out/bench.err
DG_TILE_NNZ=1048576 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_t1m.json 2>>gpurun_out/bench.err
python bench.py --no-cpu-baseline --steps 10 --accum fp32 > gpurun_out/bench_fp32.json 2>>gpurun_out/bench.err
bash scripts/gpu_prof.sh k_tiles 1 tiles4_w0
