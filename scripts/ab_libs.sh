# Interleaved same-box A/B of alternative builds: ablibs/lib_<v>.so swapped into place.
# usage: LIBS="old new" REPS=3 ARGS="--steps 30" bash scripts/ab_libs.sh
mkdir -p gpurun_out
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt_fp32') or {}; print(round(d['ms_per_step'],4), 'kern', {k: round(v['ms'],4) for k, v in d['roofline']['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],4), 'fp32', round(a.get('ms_per_step',0),4))"; }
cp paper_2103_09683_b200/libdosegpu.so /tmp/lib_current.so
{
for r in $(seq ${REPS:-3}); do
  for v in ${LIBS}; do
    cp ablibs/lib_$v.so paper_2103_09683_b200/libdosegpu.so
    echo "=== [$r] $v $ARGS"; env ${ENVS} timeout 240 python bench.py --no-cpu-baseline $ARGS | q
  done
done
} > gpurun_out/${OUT:-ab_libs}.txt 2>&1
cp /tmp/lib_current.so paper_2103_09683_b200/libdosegpu.so
cat gpurun_out/${OUT:-ab_libs}.txt
