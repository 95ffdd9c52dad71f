timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "overlap or contiguous or dense" 2>&1 | tail -1
VARS="DG_D2H_STREAMS=1|DG_D2H_STREAMS=2" REPS=3 ARGS="--steps 20 --no-alt-fp32" OUT=ab_d2h bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_d2h.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
for v in 1 2; do DG_D2H_STREAMS=$v TAG=streams=$v python scripts/e2e_probe.py 2>&1 | tail -1; done
