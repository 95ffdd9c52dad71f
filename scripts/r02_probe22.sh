VARS="DG_RUNS_PER_WARP=2|DG_RUNS_PER_WARP=1|DG_TILE_GUIDE=1" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_rpw_c2 bash scripts/ab_alt.sh > /dev/null
VARS="DG_RUNS_PER_WARP=2|DG_RUNS_PER_WARP=1|DG_TILE_GUIDE=1" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_rpw_shard bash scripts/ab_alt.sh > /dev/null
VARS="DG_RUNS_PER_WARP=2|DG_RUNS_PER_WARP=1" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_rpw_c4 bash scripts/ab_alt.sh > /dev/null
for f in ab_rpw_c2 ab_rpw_shard ab_rpw_c4; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
