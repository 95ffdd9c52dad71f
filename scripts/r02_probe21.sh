VARS="DG_DENSE_ORDER=len|DG_DENSE_ORDER=cls|DG_DENSE_ORDER=cls DG_VALUES_CFG=1" REPS=2 ARGS="--steps 20 --accum fp32 --no-alt-fp32" OUT=ab_fp32 bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_fp32.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
