# slice-kernel knobs on the C3 shard (1M rows of C2)
VARS="DG_NONE=0|DG_REPLICAS=0|DG_TILE_GUIDE=1|DG_TILE_GUIDE_MIN=262144|DG_TILE_NNZ=1572864|DG_RUNS_PER_WARP=1|DG_RUNS_PER_WARP=3|DG_PDL=0" REPS=2 \
  ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_shard2 bash scripts/ab_alt.sh
