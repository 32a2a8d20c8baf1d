# A/B: merge-kernel launch bounds (transient + gated), plain-deposit register cap
V=paper_2605_11536_b200/_native/variants
O=gpurun_out/r02q; mkdir -p $O
for lib in default app5 app6 app8; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in c2r t1080b64 c3w c3; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$lib.json 2>/dev/null
  done
done
for i in 1 2; do
for lib in default plain3 plain5 phist; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in c4p c2p; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_${lib}_$i.json 2>/dev/null
  done
done
done
unset TOFR_B200_LIB
bash tools/gpu_run.sh r02q kprof:c4p:k_hist_plain:1:25 > /dev/null 2>&1
