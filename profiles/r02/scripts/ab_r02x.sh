O=gpurun_out/r02x; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -k "transient or sparse or full_size or sessions or plain or bands" > $O/tests.log 2>&1; tail -2 $O/tests.log
V=paper_2605_11536_b200/_native/variants
for lib in default nobincache; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in t1080b64 c2r t1080; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$lib.json 2>/dev/null
  done
  python bench.py --workload c4r --steps 10 --warmup 25 --no-cpu-baseline > $O/c4r_$lib.json 2>/dev/null
done
unset TOFR_B200_LIB
bash tools/gpu_run.sh r02x kprof:t1080b64:k_trace_bins:1:25 > /dev/null 2>&1
