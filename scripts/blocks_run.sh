# Output row-block count (address locality of a tile's segments) on C2 and C5.  gpurun_out/blocks.txt
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['value']), 'e2e', round(d['e2e']['ms_per_step'],4), 'setup', d['config']['setup_s'], {k: v['ms'] for k, v in d['roofline']['kernels'].items()})"; }
{
for b in 8 32 64; do
  echo "=== c2 DG_BLOCKS=$b"; DG_BLOCKS=$b timeout 600 python bench.py --no-cpu-baseline --no-alt-fp32 --steps 30 | q
done
for b in 8 64; do
  echo "=== c5 DG_BLOCKS=$b"; DG_BLOCKS=$b timeout 900 python bench.py --config c5 --no-cpu-baseline --steps 5 | q
done
} > gpurun_out/blocks.txt 2>&1
cat gpurun_out/blocks.txt
