#!/bin/bash
# A/B of chunked path-tree CTAs (TOFR_TRACE_CHUNK pixels per CTA, 0 = persistent CTAs): a side-stream
# initial sampling made of short-lived CTAs hands SM slots back to the session stream between chunks
O=gpurun_out/ab_chunk; mkdir -p $O
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernel_ms_per_step',{}); print(round(d['value'],2), round(d['e2e']['value'],2), k.get('k_trace_gated', k.get('k_trace_bins')))" $1; }
for wl in ${WLS:-c3 c3w c1 nlos t1080b64 c3}; do
  for ch in 0 512 2048; do
    TOFR_TRACE_CHUNK=$ch timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$ch.json 2> $O/$wl.$ch.err
    echo "$wl chunk=$ch $(val $O/$wl.$ch.json)" | tee -a $O/summary.txt
  done
done
