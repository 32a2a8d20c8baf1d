#!/bin/bash
# A/B of library variants without the test suite: bash tools/gpu_var.sh <tag> "<workloads>" variant...
TAG=$1; WLS=$2; shift 2
O=gpurun_out/$TAG; mkdir -p $O
for v in "$@"; do
  for wl in $WLS; do
    case $v in
      default) env="" ;;
      *) env="TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_$v.so" ;;
    esac
    env $env timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${v}_$wl.json 2> $O/bench_${v}_$wl.err
    python -c "import json; d=json.load(open('$O/bench_${v}_$wl.json')); print('$v $wl', round(d['value'],2), d['stage_ms'])" 2>/dev/null || { echo "$v $wl FAILED"; tail -3 $O/bench_${v}_$wl.err; }
  done
done
