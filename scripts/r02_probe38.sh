VARS="DG_NONE=0|DG_TILE_GUIDE_MIN=32768|DG_TILE_GUIDE_MIN=16384|DG_TILE_GUIDE=1|DG_TILE_GUIDE=1 DG_TILE_GUIDE_MIN=32768" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_gm_shard bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_gm_shard.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
