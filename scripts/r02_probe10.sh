# C2 end to end: overlapped download granularity
VARS="DG_NONE=0|DG_NO_OVERLAP=1|DG_BLOCKS=8|DG_BLOCKS=16|DG_BLOCKS=64|DG_PDL=0" REPS=2 ARGS="--steps 20 --no-alt-fp32" OUT=ab_e2e bash scripts/ab_alt.sh > /dev/null
grep -A1 "===" gpurun_out/ab_e2e.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/'
