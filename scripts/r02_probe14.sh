timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
LIBS="p2 trim" REPS=3 ARGS="--steps 20" OUT=ab_trim_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="p2 trim" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_trim_shard bash scripts/ab_libs.sh > /dev/null
LIBS="p2 trim" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_trim_c4 bash scripts/ab_libs.sh > /dev/null
for f in ab_trim_c2 ab_trim_shard ab_trim_c4; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
