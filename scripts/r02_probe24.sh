timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -2
VARS="DG_VALUES_AFTER=0|DG_VALUES_AFTER=1" REPS=3 ARGS="--steps 20" OUT=ab_va_c2 bash scripts/ab_alt.sh > /dev/null
VARS="DG_VALUES_AFTER=0|DG_VALUES_AFTER=1" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_va_shard bash scripts/ab_alt.sh > /dev/null
VARS="DG_VALUES_AFTER=0|DG_VALUES_AFTER=1" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_va_c1 bash scripts/ab_alt.sh > /dev/null
for f in ab_va_c2 ab_va_shard ab_va_c1; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
