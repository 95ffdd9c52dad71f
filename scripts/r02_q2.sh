set -x
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_ddm_io.py tests/test_multi_gpu.py -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/q_bench.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print(d['ms_per_step'],d['roofline']['kernels'],d['e2e']['ms_per_step'],d['alt_fp32']['ms_per_step'])"
ncu --clock-control none -k regex:"k_(slices|dense|tiles)" -s 2 -c 2 --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 2>&1 | grep -E "  k_|gpu__|dram|l1tex|smsp" | cut -c1-150
DG_TRACE=1 timeout 300 python scripts/trace_tiles.py --rows 1000000 2>&1 | tail -25
bash scripts/sanitize.sh
