LIBS="carry20 carry24 carry32" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_carry bash scripts/ab_libs.sh > /dev/null
grep -A1 "===" gpurun_out/ab_carry.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
