# ncu --set full of the C2 tile kernel (and k_dense) -> gpurun_out/r02_<tag>.ncu-rep
TAG=${TAG:-tiles}
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_tiles}" -s ${SKIP:-3} -c 1 \
    -o gpurun_out/r02_$TAG -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline $ARGS > gpurun_out/r02_$TAG.log 2>&1
tail -2 gpurun_out/r02_$TAG.log
