#!/bin/bash
# round-1 GPU session: parity tests, bench lines, launch list, one full ncu capture
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
(nproc; lscpu | grep -E "Model name|^CPU\(s\)") > gpurun_out/host.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --workload c3w --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3w.json 2>&1
timeout 300 python bench.py --workload c1 --steps 20 --warmup 3 > gpurun_out/bench_c1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spatial -s 3 -c 1 \
    -o gpurun_out/prof_spatial_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_init_gated -s 3 -c 1 \
    -o gpurun_out/prof_init_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_init.log 2>&1
ls -la gpurun_out
