LIBS="p2 p3 p4" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_p_c4 bash scripts/ab_libs.sh > /dev/null
LIBS="p2 p3 p4" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_p_c2 bash scripts/ab_libs.sh > /dev/null
for f in ab_p_c4 ab_p_c2; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
