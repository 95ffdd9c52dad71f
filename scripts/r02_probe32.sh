timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
DG_SHORT_SEGMENTS=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
LIBS="w32 mix" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_mix_c1 bash scripts/ab_libs.sh > /dev/null
LIBS="w32 mix" REPS=2 ARGS="--steps 20" OUT=ab_mix_c2 bash scripts/ab_libs.sh > /dev/null
LIBS="w32 mix" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_mix_c4 bash scripts/ab_libs.sh > /dev/null
for f in ab_mix_c1 ab_mix_c2 ab_mix_c4; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
