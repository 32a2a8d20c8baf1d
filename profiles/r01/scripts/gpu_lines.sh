#!/bin/bash
# Bench lines of every workload (no profiler): bash tools/gpu_lines.sh <tag>
TAG=${1:-lines}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log | cut -c1-60
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for wl in c3w c3d c5 c1 c2p c2r c4p; do
  timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 900 python bench.py --workload c4r --steps 10 --warmup 3 > $O/bench_c4r.json 2> $O/bench_c4r.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for f in $O/bench_*.json; do python -c "
import json,sys
d=json.load(open('$f'))
if d.get('impl'): print('$f', d.get('value')); sys.exit()
print('$f'.split('/')[-1], round(d['value'],2), 'e2e', round(d['e2e']['value'],2), (d.get('frame_latency') or {}).get('p50_ms'))
"; done
