#!/bin/bash
# A/B of the three-frame pipeline (gated sessions; TOFR_PIPE_DEPTH=2: two frames), same box, interleaved
O=gpurun_out/ab_pipe; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "pipelined or sessions or bands or parity_gated or fullsize" > $O/pytest.log 2>&1; tail -2 $O/pytest.log | tee -a $O/summary.txt
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['e2e']['value'],2))" $1; }
for wl in ${WLS:-c3 c3w nlos c1 c3d c3 mesh}; do
  for dp in 2 3; do
    TOFR_PIPE_DEPTH=$dp timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$dp.json 2> $O/$wl.$dp.err
    echo "$wl depth=$dp $(val $O/$wl.$dp.json)" | tee -a $O/summary.txt
  done
done
