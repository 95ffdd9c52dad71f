# C4: overlapped host download for fused multi-wave plans, wave lag / block count
LIBS="base ovl" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_c4_ovl bash scripts/ab_libs.sh > /dev/null
VARS="DG_WAVE_LAG=1|DG_WAVE_LAG=2|DG_WAVE_LAG=4|DG_BLOCKS=32 DG_WAVE_LAG=4|DG_BLOCKS=32 DG_WAVE_LAG=8|DG_BLOCKS=32" REPS=1 ARGS="--steps 10 --config c4 --no-alt-fp32" OUT=ab_c4_lag bash scripts/ab_alt.sh > /dev/null
for f in ab_c4_ovl ab_c4_lag; do echo "## $f"; grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'; done
