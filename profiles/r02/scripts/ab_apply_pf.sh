O=gpurun_out/ab_apf; mkdir -p $O
V=paper_2605_11536_b200/_native/variants
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or sparse or transient or fullsize" > $O/pytest.log 2>&1; tail -1 $O/pytest.log | tee -a $O/summary.txt
for wl in t1080b64 c2r c3 t1080b64 c2r; do for lib in main pf0; do
  if [ $lib = main ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$lib.json 2> $O/$wl.$lib.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); k=d.get('kernel_ms_per_step',{}); print(sys.argv[2], round(d['value'],2), round(d['e2e']['value'],2), k.get('k_temporal_apply'))" $O/$wl.$lib.json "$wl $lib" | tee -a $O/summary.txt
done; done
