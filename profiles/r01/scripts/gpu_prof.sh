#!/bin/bash
# Launch lists + one full ncu capture of the named kernels.
#   bash tools/gpu_prof.sh <tag> <workload> "<kernel regex>" [skip] [count]
TAG=$1; WL=$2; RX=$3; SKIP=${4:-40}; CNT=${5:-4}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$WL.csv \
    python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch_$WL.log 2>&1
python tools/ncu_summary.py launches $O/launches_$WL.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c $CNT -o $O/prof_$WL \
    python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_$WL.log 2>&1
python tools/ncu_summary.py full $O/prof_$WL.ncu-rep
