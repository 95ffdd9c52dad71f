LIBS="w32 w28 w24" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_w_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="w32 w28" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_w_shard bash scripts/ab_libs.sh > /dev/null
for f in ab_w_c2 ab_w_shard; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
