timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "split or wave or multibeam or million or dense or edge" 2>&1 | tail -2
LIBS="base peek" REPS=2 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_peek_c4 bash scripts/ab_libs.sh > /dev/null
grep -A1 "===" gpurun_out/ab_peek_c4.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
