timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
LIBS="base reuse" REPS=3 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_reuse_c1 bash scripts/ab_libs.sh > /dev/null
LIBS="base reuse" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_reuse_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="base reuse" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_reuse_shard bash scripts/ab_libs.sh > /dev/null
for f in ab_reuse_c1 ab_reuse_c2 ab_reuse_shard; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
