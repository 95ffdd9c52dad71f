VARS="DG_NONE=0|DG_RUNS_PER_WARP=1|DG_RUNS_PER_WARP=3|DG_TILE_NNZ=524288|DG_TILE_NNZ=1048576" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_k28_c2 bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_k28_c2.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
