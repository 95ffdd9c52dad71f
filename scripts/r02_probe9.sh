timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "contiguous or dense or edge" 2>&1 | tail -3
VARS="DG_VALUES_CFG=0|DG_VALUES_CFG=1|DG_VALUES_CFG=2|DG_VALUES_CFG=3" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_vcfg bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_vcfg.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
