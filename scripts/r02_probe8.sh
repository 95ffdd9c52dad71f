# value-only contiguous rows: full GPU suite, then base/vals A/B on C2, shard, C5-sized check
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
LIBS="base vals" REPS=2 ARGS="--steps 20" OUT=ab_vals_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="base vals" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_vals_shard bash scripts/ab_libs.sh > /dev/null
for f in ab_vals_c2 ab_vals_shard; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
