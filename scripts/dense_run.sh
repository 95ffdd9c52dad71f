# Dense-row kernel A/B on C2, its 1/8 shard, and C4.  Output gpurun_out/dense.txt
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt_fp32') or {}; print(round(d['ms_per_step'],4), round(d['value']), 'kern', {k: v['ms'] for k, v in d['roofline']['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],4), 'fp32', round(a.get('ms_per_step',0),4))"; }
{
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for v in ${VARS:-"DG_DENSE=0" "DG_DENSE_CONCURRENT=0" "DG_DENSE_CONCURRENT=1"}; do
  echo "=== c2 $v"; env $v timeout 180 python bench.py --no-cpu-baseline --steps 30 | q
  echo "=== shard(1M rows) $v"; env $v timeout 180 python bench.py --no-cpu-baseline --steps 30 --rows 1000000 | q
done
echo "=== c4"; timeout 300 python bench.py --config c4 --no-cpu-baseline --no-alt-fp32 --steps 20 | q
} > gpurun_out/dense.txt 2>&1
cat gpurun_out/dense.txt
