timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
DG_SHORT_SEGMENTS=1 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py -x -q -m gpu 2>&1 | tail -1
VARS="DG_SHORT_SEGMENTS=0|DG_SHORT_SEGMENTS=1" REPS=3 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_u4_c1 bash scripts/ab_alt.sh > /dev/null
VARS="DG_SHORT_SEGMENTS=0|DG_SHORT_SEGMENTS=1" REPS=1 ARGS="--steps 20 --no-alt-fp32" OUT=ab_u4_c2 bash scripts/ab_alt.sh > /dev/null
for f in ab_u4_c1 ab_u4_c2; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
