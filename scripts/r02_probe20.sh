VARS="DG_NONE=0|DG_TILE_NNZ=131072|DG_TILE_NNZ=262144|DG_TILE_NNZ=524288|DG_SHORT_MAX=32|DG_RUNS_PER_WARP=1" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_c1 bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_c1.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
