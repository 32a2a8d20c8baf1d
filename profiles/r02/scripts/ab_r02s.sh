O=gpurun_out/r02s; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout 1200 -k "sparse or full_size or bands or sessions" > $O/tests.log 2>&1; tail -2 $O/tests.log
for a in 1 0; do
  for wl in t1080b64 t1080 c2r; do
    TOFR_ADAPTIVE_BATCHES=$a python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$a.json 2>/dev/null
  done
  TOFR_ADAPTIVE_BATCHES=$a python bench.py --workload c4r --steps 10 --warmup 25 --no-cpu-baseline > $O/c4r_$a.json 2>/dev/null
done
