#!/bin/bash
# phased spatial pass vs monolithic k_spatial; band parity; C++ shim; ncu of the phased kernels
mkdir -p gpurun_out/r01d
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r01d/pytest_gpu.log 2>&1
run() { timeout 300 python bench.py --workload $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01d/bench_$1_$2.json 2>&1; }
for wl in c3 c3w c1; do
  TOFR_SPATIAL=mono run mono $wl
  run phased $wl
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d/launches_c3w.csv \
    python bench.py --workload c3w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01d/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial_ -s 10 -c 5 \
    -o gpurun_out/r01d/prof_phased_c3w python bench.py --workload c3w --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r01d/ncu.log 2>&1
