#!/bin/bash
# One full ncu capture (with source) of one kernel launch, exported for tools/ncu_lines.py.
#   bash tools/gpu_src.sh <tag> <workload> <kernel regex> <skip>
TAG=$1; WL=$2; RX=$3; SKIP=${4:-20}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$RX" -s $SKIP -c 1 -o $O/src_$WL \
    python bench.py --workload $WL --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_src_$WL.log 2>&1
python tools/ncu_summary.py full $O/src_$WL.ncu-rep
