#!/bin/bash
# persistent CTAs with dynamic warp work distribution
mkdir -p gpurun_out/r01f
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01f/pytest_gpu.log 2>&1
run() { timeout 300 python bench.py --workload $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01f/bench_$1_$2.json 2>&1; }
for wl in c3 c3w c1 c5; do run dyn $wl; done
TOFR_ORDER=0 run dyn_o0 c3w
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01f/launches_c3.csv \
    python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01f/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial_fwd$ -s 3 -c 1 \
    -o gpurun_out/r01f/prof_fwd_c3w python bench.py --workload c3w --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/r01f/ncu.log 2>&1
