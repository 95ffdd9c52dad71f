LIBS="p2 p3" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_p28_c4 bash scripts/ab_libs.sh > /dev/null
LIBS="p2 p3" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_p28_c1 bash scripts/ab_libs.sh > /dev/null
for f in ab_p28_c4 ab_p28_c1; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
