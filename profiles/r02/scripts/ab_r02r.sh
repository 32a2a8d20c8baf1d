# A/B: finish launch bounds (transient), plain 6 CTAs, apply 6; nlos_scan; ncu of the new plain kernel
V=paper_2605_11536_b200/_native/variants
O=gpurun_out/r02r; mkdir -p $O
for lib in default fin5 fin6 app6; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in c2r t1080b64 c3; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$lib.json 2>/dev/null
  done
done
for lib in default plain6; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in c4p c2p; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$lib.json 2>/dev/null
  done
done
unset TOFR_B200_LIB
python bench.py --workload nlos_scan --steps 20 --warmup 25 > $O/nlos_scan.json 2> $O/nlos_scan.err
python bench.py --workload nlos --steps 20 --warmup 25 --no-cpu-baseline > $O/nlos.json 2>/dev/null
bash tools/gpu_run.sh r02r kprof:c4p:k_hist_plain:1:25 kprof:c2p:k_hist_plain:1:25 > /dev/null 2>&1
