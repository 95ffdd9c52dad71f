# quick GPU check: parity tests + C2 A/B replicas off/on
set -x
python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -15
VARS="DG_REPLICAS=0|DG_REPLICAS=1" REPS=2 ARGS="--steps 20 --warmup 5" bash scripts/ab_alt.sh
