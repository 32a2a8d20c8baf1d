#!/bin/bash
# outlined FP64 div/sqrt vs inline; parity suite after the phased spatial pass
mkdir -p gpurun_out/r01e
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01e/pytest_gpu.log 2>&1
run() { timeout 300 python bench.py --workload $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01e/bench_$1_$2.json 2>&1; }
for wl in c3 c3w; do
  run outl $wl
  TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_inl.so run inl $wl
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial_fwd -s 3 -c 2 \
    -o gpurun_out/r01e/prof_fwd_c3w python bench.py --workload c3w --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r01e/ncu.log 2>&1
