#!/bin/bash
# A/B of library variants: GPU tests on the default build, then bench lines per variant.
#   bash tools/gpu_ab.sh <tag> "<workloads>" [variant ...]   (variant: default | legacy | <tag of _native/variants>)
TAG=$1; WLS=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
for v in "$@"; do
  for wl in $WLS; do
    case $v in
      default) env="" ;;
      legacy) env="TOFR_REUSE=legacy" ;;
      *) env="TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_$v.so" ;;
    esac
    env $env timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${v}_$wl.json 2> $O/bench_${v}_$wl.err
    python -c "import json,sys; d=json.load(open('$O/bench_${v}_$wl.json')); print('$v $wl', round(d['value'],2), d['unit'], d['stage_ms'], 'sp', d['shift_stats_one_frame']['spatial']['attempts'])" 2>/dev/null || { echo "$v $wl FAILED"; tail -3 $O/bench_${v}_$wl.err; }
  done
done
