#!/bin/bash
# A/B of the temporal prep's items per thread (TOFR_PREP_ITEMS: main = 4, prep1 = 1, prep8 = 8)
O=gpurun_out/ab_prep; mkdir -p $O
V=paper_2605_11536_b200/_native/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or wave or sparse or sessions or fullsize or bands" > $O/pytest.log 2>&1; tail -1 $O/pytest.log | tee -a $O/summary.txt
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernel_ms_per_step',{}); print(round(d['value'],2), round(d['e2e']['value'],2), k.get("k_spatial_prep_inv"), k.get("k_spatial_prep_fwd"))" $1; }
for wl in ${WLS:-c3 c3w c1 nlos c3d c3}; do
  for lib in main prep1; do
    if [ $lib = main ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
    timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$lib.json 2> $O/$wl.$lib.err
    echo "$wl $lib $(val $O/$wl.$lib.json)" | tee -a $O/summary.txt
  done
done
unset TOFR_B200_LIB
timeout 900 python bench.py --workload c4r --steps 6 --warmup 25 --no-cpu-baseline > $O/c4r.main.json 2>&1; TOFR_B200_LIB=$V/libtofr_b200_prep1.so timeout 900 python bench.py --workload c4r --steps 6 --warmup 25 --no-cpu-baseline > $O/c4r.prep1.json 2>&1; for l in main prep1; do echo "c4r $l $(val $O/c4r.$l.json)" | tee -a $O/summary.txt; done
