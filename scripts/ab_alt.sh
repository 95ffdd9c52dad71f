# Interleaved same-box A/B (box-to-box variance is ~5%): VARS alternated REPS times.
# usage: VARS="DG_DENSE=0|DG_DENSE=1" REPS=3 ARGS="--steps 30" bash scripts/ab_alt.sh
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt_fp32') or {}; print(round(d['ms_per_step'],4), 'kern', {k: round(v['ms'],4) for k, v in d['roofline']['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],4), 'fp32', round(a.get('ms_per_step',0),4))"; }
IFS='|' read -ra VS <<< "${VARS}"
{
for r in $(seq ${REPS:-3}); do
  for v in "${VS[@]}"; do
    echo "=== [$r] $v $ARGS"; env $v timeout 240 python bench.py --no-cpu-baseline $ARGS | q
  done
done
} > gpurun_out/${OUT:-ab_alt}.txt 2>&1
cat gpurun_out/${OUT:-ab_alt}.txt
