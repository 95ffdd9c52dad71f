LIBS="old st stpad8 pad8 new" ENVS="DG_RUNS_PER_WARP=1" REPS=2 ARGS="--steps 20 --no-alt-fp32" bash scripts/ab_libs.sh
