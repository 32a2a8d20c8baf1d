#!/bin/bash
# Quick iteration on the GPU box: GPU test suite + bench lines for the given workloads.
#   bash tools/gpu_quick.sh <tag> [workload ...]
TAG=${1:-quick}; shift
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
for wl in "${@:-c3}"; do
  timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
  python -c "import json,sys; d=json.load(open('$O/bench_$wl.json')); print('$wl', round(d['value'],2), d['unit'], d['stage_ms'], 'e2e', round(d['e2e']['value'],2))" || tail -5 $O/bench_$wl.err
done
