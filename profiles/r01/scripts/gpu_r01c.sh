#!/bin/bash
# cost-ordered reuse kernels (TOFR_ORDER) x register caps; band parity on GPU; ncu of k_spatial
mkdir -p gpurun_out/r01c
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01c/pytest_gpu.log 2>&1
run() { timeout 300 python bench.py --workload $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01c/bench_$1_$2.json 2>&1; }
for wl in c3 c3w; do
  TOFR_ORDER=0 run m4o0 $wl
  run m4 $wl
  TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_m3.so run m3 $wl
  TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_m5.so run m5 $wl
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spatial -s 3 -c 1 \
    -o gpurun_out/r01c/prof_spatial_c3w python bench.py --workload c3w --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01c/ncu.log 2>&1
