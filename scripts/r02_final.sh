# final check on HEAD: GPU suite, smoke, C2 headline (driver-style) twice, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.txt 2>&1; tail -n 2 gpurun_out/gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1; tail -n 2 gpurun_out/smoke.txt
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2_20_$i.json 2> gpurun_out/bench_c2_20.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_c2_20_$i.json').read().strip().splitlines()[-1]); print('c2', d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -c 400 gpurun_out/bench_reference.json
