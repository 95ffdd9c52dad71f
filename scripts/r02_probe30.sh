timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
LIBS="w32 w28b" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_w_c1 bash scripts/ab_libs.sh > /dev/null
LIBS="w32 w28b" REPS=2 ARGS="--steps 20 --accum fp32 --no-alt-fp32" OUT=ab_w_fp32 bash scripts/ab_libs.sh > /dev/null
LIBS="w32 w28b" REPS=1 ARGS="--steps 5 --config c5 --no-alt-fp32" OUT=ab_w_c5 bash scripts/ab_libs.sh > /dev/null
for f in ab_w_c1 ab_w_fp32 ab_w_c5; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
