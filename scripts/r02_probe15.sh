timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu 2>&1 | tail -2
LIBS="base vlast" REPS=3 ARGS="--steps 20" OUT=ab_vlast bash scripts/ab_libs.sh > /dev/null
LIBS="base vlast" REPS=2 ARGS="--steps 30 --rows 1000000 --no-alt-fp32" OUT=ab_vlast_shard bash scripts/ab_libs.sh > /dev/null
for f in ab_vlast ab_vlast_shard; do grep -A1 "===" gpurun_out/$f.txt | grep -v "^--" | paste - - | sed -E 's/--steps.*fp32 *\t/\t/; s/--steps 20\t/\t/'; done
