# Tile-timeline traces of C2 under plan variants (DG_* knobs); output gpurun_out/trace_c2.txt
mkdir -p gpurun_out
for v in "DG_TILE_GUIDE=0" "DG_TILE_GUIDE=2" "DG_TILE_GUIDE=3" "DG_TILE_GUIDE=2 DG_TILE_GUIDE_MIN=131072" "DG_TILE_GUIDE=4 DG_TILE_GUIDE_MIN=32768"; do
  echo "=== exact $v" ; env $v timeout 300 python scripts/trace_tiles.py --config c2 | grep -v "in flight"
done > gpurun_out/trace_c2.txt 2>&1
echo "=== fp32" >> gpurun_out/trace_c2.txt
timeout 300 python scripts/trace_tiles.py --config c2 --accum fp32 | grep -v "in flight" >> gpurun_out/trace_c2.txt 2>&1
for v in "DG_TILE_GUIDE=0" "DG_TILE_GUIDE=2" "DG_TILE_GUIDE=3"; do
  echo "=== bench $v"; env $v timeout 300 python bench.py --no-cpu-baseline --steps 30 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['alt_fp32']['ms_per_step'], d['e2e']['ms_per_step'])"
done >> gpurun_out/trace_c2.txt 2>&1
cat gpurun_out/trace_c2.txt
