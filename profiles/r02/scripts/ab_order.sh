#!/bin/bash
# A/B of the slow-first solve order (TOFR_SOLVE_ORDER=0: queue order), same box, interleaved
O=gpurun_out/ab_order; mkdir -p $O
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d.get('kernel_ms_per_step',{}).get('k_shift_solve'))" $1; }
for wl in ${WLS:-c3 c3w nlos c1 t1080b64}; do
  for rep in 1 2; do
    for o in 0 1; do
      TOFR_SOLVE_ORDER=$o timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$o.$rep.json 2> $O/$wl.$o.$rep.err
      echo "$wl order=$o rep=$rep $(val $O/$wl.$o.$rep.json)" | tee -a $O/summary.txt
    done
  done
done
for o in 0 1; do
  TOFR_SOLVE_ORDER=$o timeout 900 python tools/band_probe2.py c3 8 > $O/band_c3_8.$o.log 2>&1
  echo "band c3 8 order=$o"; cat $O/band_c3_8.$o.log
done | tee -a $O/summary.txt
