LIBS="old onest one" ENVS="DG_RUNS_PER_WARP=1" REPS=2 ARGS="--steps 20 --no-alt-fp32" bash scripts/ab_libs.sh
LIBS="one" ENVS="DG_RUNS_PER_WARP=2" REPS=2 ARGS="--steps 20" bash scripts/ab_libs.sh
LIBS="old one" ENVS="DG_RUNS_PER_WARP=2" REPS=2 ARGS="--steps 30 --no-alt-fp32 --rows 1000000" bash scripts/ab_libs.sh
