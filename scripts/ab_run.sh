# A/B of tile-kernel configs on C2 (exact + fp32) after a kernel change.  gpurun_out/ab.txt
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt_fp32') or {}; print(round(d['ms_per_step'],4), round(d['value']), 'kern', {k: v['ms'] for k, v in d['roofline']['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],4), 'fp32', round(a.get('ms_per_step',0),4))"; }
{
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in ${CFGS:-0 8 10}; do
  echo "=== c2 cfg $c"; DG_TILE_CFG=$c timeout 600 python bench.py --no-cpu-baseline --steps 30 | q
done
} > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
