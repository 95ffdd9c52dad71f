#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.txt

DG_TILE_CFG=9 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1 or desk or wide" 2>&1 | tail -3 >> gpurun_out/gpu_tests.txt
for c in 0 8 9 10; do
  DG_TILE_CFG=$c python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg$c.json 2>>gpurun_out/bench.err
  DG_TILE_CFG=$c python bench.py --no-cpu-baseline --steps 10 --accum fp32 > gpurun_out/bench_f32_cfg$c.json 2>>gpurun_out/bench.err
done
DG_TILE_CFG=9 bash scripts/gpu_prof.sh k_tiles 1 pf9
