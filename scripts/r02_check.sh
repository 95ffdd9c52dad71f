# quick GPU check: parity tests + C2 A/B
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -25
VARS="${VARS:-DG_SLICES=0|DG_SLICES=1}" REPS=${REPS:-2} ARGS="--steps 20 --warmup 5" bash scripts/ab_alt.sh
