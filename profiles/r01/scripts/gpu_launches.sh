#!/bin/bash
# ncu launch lists (gpu__time_duration per kernel) of several workloads.
#   bash tools/gpu_launches.sh <tag> <workload> ...
TAG=$1; shift
O=gpurun_out/$TAG
mkdir -p $O
for WL in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$WL.csv \
      python bench.py --workload $WL --steps 4 --warmup 3 --no-cpu-baseline > $O/ncu_launch_$WL.log 2>&1
  echo "== $WL"; python tools/ncu_summary.py launches $O/launches_$WL.csv
done
