#!/bin/bash
# transient workloads (plain + reservoir), pipelined e2e, full suite
mkdir -p gpurun_out/r01g
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01g/pytest_gpu.log 2>&1
run() { timeout 400 python bench.py --workload $2 --steps 10 --warmup 3 $3 > gpurun_out/r01g/bench_$1_$2.json 2>&1; }
run a c3
for wl in c2p c2r c4p; do run a $wl --no-cpu-baseline; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01g/launches_c2r.csv \
    python bench.py --workload c2r --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01g/ncu_launch.log 2>&1
