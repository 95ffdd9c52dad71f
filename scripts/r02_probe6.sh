# warp-collective refill + static first tiles: parity, then old/new A/B (shard, C2)
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
LIBS="old new" REPS=3 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_refill_shard bash scripts/ab_libs.sh > /dev/null
LIBS="old new" REPS=2 ARGS="--steps 20" OUT=ab_refill_c2 bash scripts/ab_libs.sh > /dev/null
ENVS="DG_TILE_GUIDE=1 DG_RUNS_PER_WARP=1" LIBS="old new" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_refill_shard_g1r1 bash scripts/ab_libs.sh > /dev/null
for f in ab_refill_shard ab_refill_c2 ab_refill_shard_g1r1; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
