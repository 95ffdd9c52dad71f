VARS="DG_DENSE_CLASS=0|DG_DENSE_CLASS=1|DG_DENSE_CLASS=2" REPS=3 ARGS="--steps 20 --no-alt-fp32" OUT=ab_class bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_class.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
