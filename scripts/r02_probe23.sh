VARS="DG_TILES_PER_SM=8|DG_TILES_PER_SM=4|DG_TILES_PER_SM=2|DG_TILES_PER_SM=4 DG_TILE_GUIDE=1" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_tps_shard bash scripts/ab_alt.sh > /dev/null
VARS="DG_TILES_PER_SM=8|DG_TILES_PER_SM=4" REPS=2 ARGS="--steps 30 --rows 2000000 --no-alt-fp32" OUT=ab_tps_shard4 bash scripts/ab_alt.sh > /dev/null
VARS="DG_TILES_PER_SM=8|DG_TILES_PER_SM=4" REPS=2 ARGS="--steps 30 --config c1 --no-alt-fp32" OUT=ab_tps_c1 bash scripts/ab_alt.sh > /dev/null
for f in ab_tps_shard ab_tps_shard4 ab_tps_c1; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
