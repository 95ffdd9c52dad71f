timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_fullscale_gpu.py -x -q -m gpu -k "not c5 and not c4_full and not shards" 2>&1 | tail -1
LIBS="nofma fma" REPS=2 ARGS="--steps 20" OUT=ab_fma bash scripts/ab_libs.sh > /dev/null
grep -A1 "===" gpurun_out/ab_fma.txt | grep -v "^--" | paste - - | sed -E 's/--steps 20\t/\t/'
