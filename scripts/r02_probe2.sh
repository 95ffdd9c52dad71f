# k_dense share A/B on the C3 shard and on C2
VARS="DG_NONE=0|DG_DENSE_MIN_LEN=1024|DG_DENSE_MIN_LEN=2048|DG_DENSE_MIN_LEN=8192|DG_DENSE_MIN_LEN=13000" REPS=2 \
  ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_shard bash scripts/ab_alt.sh
VARS="DG_NONE=0|DG_DENSE=1|DG_DENSE=1 DG_DENSE_MIN_LEN=8192" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_c2 bash scripts/ab_alt.sh
