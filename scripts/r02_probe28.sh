timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
timeout 900 python -m pytest tests/test_fullscale_gpu.py -x -q -m gpu -k "c2_full_vector" 2>&1 | tail -1
VARS="DG_VALUE_PAIRS=0|DG_VALUE_PAIRS=1" REPS=2 ARGS="--steps 20" OUT=ab_pairs bash scripts/ab_alt.sh > /dev/null
LIBS="pairs pairs4" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_pairs_minb bash scripts/ab_libs.sh > /dev/null
VARS="DG_VALUE_PAIRS=0|DG_VALUE_PAIRS=1" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_pairs_shard bash scripts/ab_alt.sh > /dev/null
for f in ab_pairs ab_pairs_minb ab_pairs_shard; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
