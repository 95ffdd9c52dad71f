# tile guide / runs per warp combinations: C3 shard, C2, C4
VARS="DG_NONE=0|DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1|DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1 DG_TILE_NNZ=1572864|DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1 DG_TILE_GUIDE_MIN=131072" REPS=2 \
  ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_shard3 bash scripts/ab_alt.sh
VARS="DG_NONE=0|DG_TILE_GUIDE=1|DG_RUNS_PER_WARP=1|DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_c2b bash scripts/ab_alt.sh
VARS="DG_NONE=0|DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_c4 bash scripts/ab_alt.sh
