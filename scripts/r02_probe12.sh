LIBS="carry24 carry26 carry28" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_carry2 bash scripts/ab_libs.sh > /dev/null
grep -A1 "===" gpurun_out/ab_carry2.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
