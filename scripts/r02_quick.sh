# quick GPU loop: parity tests, C2 bench (20 steps), a few ncu counters of the dose kernels
set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BARGS} > gpurun_out/q_bench.json 2>&1; tail -c 2200 gpurun_out/q_bench.json
ncu --clock-control none -k regex:"k_(slices|dense|tiles)" -s 2 -c 2 --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-alt-fp32 ${BARGS} 2>&1 | grep -E "k_|gpu__|dram|l1tex|smsp" | cut -c1-150
