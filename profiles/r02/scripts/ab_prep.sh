#!/bin/bash
# A/B of the temporal prep's items per thread (TOFR_PREP_ITEMS: main = 4, prep1 = 1, prep8 = 8)
O=gpurun_out/ab_prep; mkdir -p $O
V=paper_2605_11536_b200/_native/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or wave or sparse or sessions or fullsize or bands" > $O/pytest.log 2>&1; tail -1 $O/pytest.log | tee -a $O/summary.txt
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernel_ms_per_step',{}); print(round(d['value'],2), round(d['e2e']['value'],2), k.get('k_temporal_prep'))" $1; }
for wl in ${WLS:-t1080b64 c2r c3 t1080}; do
  for lib in main prep1 prep8; do
    if [ $lib = main ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
    timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$lib.json 2> $O/$wl.$lib.err
    echo "$wl $lib $(val $O/$wl.$lib.json)" | tee -a $O/summary.txt
  done
done
unset TOFR_B200_LIB
bash tools/gpu_run.sh ab_prep full:t1080b64:k_temporal_prep:200:1 > /dev/null 2>&1
