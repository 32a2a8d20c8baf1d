#!/bin/bash
# A/B by environment: bash tools/gpu_ab2.sh <tag> "<workloads>" "<NAME=VAL|default>" ...
TAG=$1; WLS=$2; shift 2
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
for v in "$@"; do
  for wl in $WLS; do
    env=""; [ "$v" != "default" ] && env="$v"
    tagv=$(echo "$v" | tr '=/' '__')
    env $env timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_${tagv}_$wl.json 2> $O/bench_${tagv}_$wl.err
    python -c "import json,sys; d=json.load(open('$O/bench_${tagv}_$wl.json')); print('$v $wl', round(d['value'],2), d['unit'], d['stage_ms'], 'e2e', round(d['e2e']['value'],2))" 2>/dev/null || { echo "$v $wl FAILED"; tail -3 $O/bench_${tagv}_$wl.err; }
  done
done
