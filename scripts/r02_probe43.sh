# C1 plan-knob sweep (configs[0], 1M x 4096): value stream on/off, tile size, replicas
mkdir -p gpurun_out
run() {  # $1 = tag, rest = env
  tag=$1; shift
  env "$@" timeout 120 python bench.py --config c1 --no-cpu-baseline --steps 50 --warmup 5 > gpurun_out/p43.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p43.json').read().strip().splitlines()[-1])
print('$tag', 'ms', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})" || tail -3 gpurun_out/p43.json
}
for i in 1 2; do
run base X=1
run dense0 DG_DENSE=0
run tnnz64k DG_TILE_NNZ=65536
run tnnz128k DG_TILE_NNZ=131072
run tps4 DG_TILES_PER_SM=4
run tps16 DG_TILES_PER_SM=16
run rep0 DG_REPLICAS=0
run dense0_tps4 DG_DENSE=0 DG_TILES_PER_SM=4
done
