# C1: where the slice kernel's 0.1 ms goes -- tile timeline, value-row threshold, one ncu capture
mkdir -p gpurun_out
timeout 300 python scripts/trace_tiles.py --config c1 2>&1 | grep -v "in flight" | tail -30
for v in "X=1" "DG_DENSE_MIN_LEN=100000" "X=1" "DG_DENSE_MIN_LEN=100000"; do
  env $v timeout 120 python bench.py --config c1 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/p44.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p44.json').read().strip().splitlines()[-1])
print('$v', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})"
done
bash scripts/gpu_prof.sh k_slices 8 c1slices --config c1
python scripts/ncu_brief.py gpurun_out/prof_c1slices.ncu-rep > gpurun_out/brief_c1slices.txt 2>&1; cat gpurun_out/brief_c1slices.txt
