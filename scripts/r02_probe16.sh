VARS="DG_DENSE_ORDER=len|DG_DENSE_ORDER=cls" REPS=3 ARGS="--steps 20" OUT=ab_order bash scripts/ab_alt.sh > /dev/null
VARS="DG_DENSE_ORDER=len|DG_DENSE_ORDER=cls" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_order_shard bash scripts/ab_alt.sh > /dev/null
for f in ab_order ab_order_shard; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
