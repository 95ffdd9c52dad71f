# C4 carry-kernel register budgets, fused vs per-wave launches.  Output gpurun_out/plan.txt
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline']['kernels'].items()})"; }
{
timeout 900 python -m pytest tests -x -q -m gpu -k "split_rows or multibeam" 2>&1 | tail -3
for c in 0 31; do for f in 0 1; do
  echo "=== c4 cfg $c fuse $f"; DG_TILE_CFG=$c DG_FUSE_WAVES=$f timeout 600 python bench.py --config c4 --no-cpu-baseline --no-alt-fp32 --steps 10 | q
done; done
} > gpurun_out/plan.txt 2>&1
cat gpurun_out/plan.txt
