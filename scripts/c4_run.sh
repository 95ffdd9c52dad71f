# Split-row (multi-wave) parity + C4 fused vs per-wave launches.  Output gpurun_out/c4.txt
mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -x -q -m gpu -k "split_rows or multibeam or overlapped or desk" 2>&1 | tail -4
for v in "DG_FUSE_WAVES=0" "DG_FUSE_WAVES=1"; do
  echo "=== c4 bench $v"; env $v timeout 600 python bench.py --config c4 --no-cpu-baseline --no-alt-fp32 --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['e2e']['ms_per_step'], d['roofline']['kernels'], d['config']['setup_s'])"
done
echo "=== c4 trace fused"; timeout 600 python scripts/trace_tiles.py --config c4 | grep -v "in flight"
} > gpurun_out/c4.txt 2>&1
cat gpurun_out/c4.txt
