timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_multi_gpu.py tests/test_fused_gather_gpu.py -x -q 2>&1 | tail -2
cat > /tmp/ab.sh <<'EOS'
q() { python -c "import json,sys; d=json.loads(sys.stdin.read()); a=d.get('alt_fp32') or {}; print(round(d['ms_per_step'],4), 'kern', {k: round(v['ms'],4) for k, v in d['roofline']['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],4), 'fp32', round(a.get('ms_per_step',0),4))"; }
for r in 1 2; do for v in 0 1; do echo "== ds=$v $ARGS"; DG_DENSE_SLICES=$v timeout 300 python bench.py --no-cpu-baseline $ARGS | q; done; done
EOS
ARGS="--steps 20" bash /tmp/ab.sh
ARGS="--steps 30 --rows 1000000" bash /tmp/ab.sh
