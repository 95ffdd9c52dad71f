#!/bin/bash
mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" python bench.py --no-cpu-baseline --no-alt-fp32 --steps 20 > gpurun_out/s_$tag.json 2>>gpurun_out/bench.err; }
run base
run k1 DG_BLOCKS=1
run t512k DG_TILE_NNZ=524288
run k1t512k DG_BLOCKS=1 DG_TILE_NNZ=524288
run t768k DG_TILE_NNZ=786432
run t1m DG_TILE_NNZ=1048576
run nb3t768k DG_TILE_CFG=12 DG_TILE_NNZ=786432
run base2
