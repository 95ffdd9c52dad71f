# values-after (volatile flag check, per-lane known-block mask): parity, then e2e breakdown A/B
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q -m gpu tests/test_parity_gpu.py -k "contiguous_rows" > gpurun_out/p42_tests.txt 2>&1; tail -n 2 gpurun_out/p42_tests.txt
timeout 900 python -m pytest -x -q -m gpu tests/test_fullscale_gpu.py -k "pinned_host" >> gpurun_out/p42_tests.txt 2>&1; tail -n 2 gpurun_out/p42_tests.txt
for i in 1 2; do
for va in 0 1; do TAG="VA=$va" DG_VALUES_AFTER=$va timeout 300 python scripts/e2e_probe.py; done
for b in 32 64; do TAG="VA=1 blocks=$b" DG_BLOCKS=$b timeout 300 python scripts/e2e_probe.py; done
done
