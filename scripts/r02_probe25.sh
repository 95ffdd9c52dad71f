VARS="DG_BLOCK_TAPER=0|DG_BLOCK_TAPER=1|DG_BLOCK_TAPER=1 DG_BLOCKS=24" REPS=3 ARGS="--steps 20 --no-alt-fp32" OUT=ab_taper bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_taper.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "overlap or contiguous or dense" 2>&1 | tail -1
