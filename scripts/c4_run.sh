# Split-row (multi-wave) parity + C4 variants.  Output gpurun_out/c4.txt
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline']['kernels'].items()})"; }
{
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for v in ${VARS:-"DG_BLOCKS=8" "DG_BLOCKS=64" "DG_BLOCKS=64 DG_WAVE_LAG=0" "DG_BLOCKS=64 DG_WAVE_LAG=3" "DG_BLOCKS=32"}; do
  echo "=== c4 $v"; env $v timeout 600 python bench.py --config c4 --no-cpu-baseline --no-alt-fp32 --steps 20 | q
done
} > gpurun_out/c4.txt 2>&1
cat gpurun_out/c4.txt
