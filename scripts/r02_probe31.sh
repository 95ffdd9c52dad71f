LIBS="w32 w28b" REPS=2 ARGS="--steps 5 --config c5 --no-alt-fp32" OUT=ab_w_c5b bash scripts/ab_libs.sh > /dev/null
LIBS="w32 w28b" REPS=2 ARGS="--steps 100 --no-alt-fp32" OUT=ab_w_c2_100 bash scripts/ab_libs.sh > /dev/null
for f in ab_w_c5b ab_w_c2_100; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
