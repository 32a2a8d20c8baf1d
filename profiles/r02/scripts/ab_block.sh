#!/bin/bash
# A/B of the solve / path-tree CTA size (64 vs 128 threads; same registers per thread, same
# resident warps): smaller CTAs hand their SM slots back in finer steps as a batch drains
O=gpurun_out/ab_block; mkdir -p $O
V=paper_2605_11536_b200/_native/variants
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernel_ms_per_step',{}); print(round(d['value'],2), round(d['e2e']['value'],2), k.get('k_shift_solve'), k.get('k_trace_gated', k.get('k_trace_bins')))" $1; }
for wl in ${WLS:-c3 c3w nlos c1 t1080b64 c3}; do
  for lib in main b64s b64st; do
    if [ $lib = main ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
    timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$lib.json 2> $O/$wl.$lib.err
    echo "$wl $lib $(val $O/$wl.$lib.json)" | tee -a $O/summary.txt
  done
done
