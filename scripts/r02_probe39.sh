VARS="DG_NONE=0|DG_TILE_GUIDE=1 DG_TILE_GUIDE_MIN=32768" REPS=3 ARGS="--steps 20 --no-alt-fp32" OUT=ab_gm_c2 bash scripts/ab_alt.sh > /dev/null
VARS="DG_NONE=0|DG_TILE_GUIDE=1 DG_TILE_GUIDE_MIN=32768" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_gm_c4 bash scripts/ab_alt.sh > /dev/null
for f in ab_gm_c2 ab_gm_c4; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
