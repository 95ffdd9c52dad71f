#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/gpu_tests.txt
DG_TILE_CFG=12 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "c1 or desk or wide or overlap" 2>&1 | tail -2 >> gpurun_out/gpu_tests.txt
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --steps 10 > gpurun_out/s_$tag.json 2>>gpurun_out/bench.err; }
run base
run nb3 DG_TILE_CFG=12
run nb4 DG_TILE_CFG=13
run g8k DG_GLOBAL_MIN_LEN=8192
run g4k DG_GLOBAL_MIN_LEN=4096
run nb3g8k DG_TILE_CFG=12 DG_GLOBAL_MIN_LEN=8192
run t512k DG_TILE_NNZ=524288
run nb3t512k DG_TILE_CFG=12 DG_TILE_NNZ=524288
run nb3t128k DG_TILE_CFG=12 DG_TILE_NNZ=131072
