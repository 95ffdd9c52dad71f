LIBS="p2 p3 p4" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_p28_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="p2 p3 p4" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_p28_shard bash scripts/ab_libs.sh > /dev/null
for f in ab_p28_c2 ab_p28_shard; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
