# C1 tile-kernel tail: guided-tail knob sweep (default for small plans: guide 1, min 32K)
mkdir -p gpurun_out
run() { tag=$1; shift
  env "$@" timeout 120 python bench.py --config c1 --no-cpu-baseline --no-alt-fp32 --steps 50 --warmup 5 > gpurun_out/p54.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/p54.json').read().strip().splitlines()[-1])
print('$tag', 'ms', round(d['ms_per_step'],4), {k: v['ms'] for k, v in d['roofline'].get('kernels', {}).items()})" || tail -2 gpurun_out/p54.json
}
for i in 1 2; do
run base X=1
run g2m16 DG_TILE_GUIDE=2 DG_TILE_GUIDE_MIN=16384
run g3m8 DG_TILE_GUIDE=3 DG_TILE_GUIDE_MIN=8192
run g2m8 DG_TILE_GUIDE=2 DG_TILE_GUIDE_MIN=8192
run g4m4 DG_TILE_GUIDE=4 DG_TILE_GUIDE_MIN=4096
run rpw3 DG_RUNS_PER_WARP=3
run rpw1 DG_RUNS_PER_WARP=1
done
