VARS="DG_NONE=0|DG_TILE_GUIDE=1|DG_TILE_GUIDE=1 DG_TILES_PER_SM=4|DG_TILE_GUIDE=1 DG_TILE_GUIDE_MIN=131072|DG_TILE_GUIDE=0|DG_TILE_GUIDE=3" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_guide_shard bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_guide_shard.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
