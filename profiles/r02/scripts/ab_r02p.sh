# A/B: slow-chain escalation variants; plain walk with history (traffic)
V=paper_2605_11536_b200/_native/variants
O=gpurun_out/r02p; mkdir -p $O
for lib in default esc2 esc3; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  for wl in c3 nlos c1 c3w; do
    python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$lib.json 2>/dev/null
  done
  python tools/band_kernels.py c3 8 7 > $O/bk87_$lib.log 2>&1
done
export TOFR_B200_LIB=$V/libtofr_b200_sprof_esc2.so; python tools/solve_profile.py c3 > $O/spc3_esc2.log 2>&1
python tools/solve_profile.py c3 8 7 > $O/sp87_esc2.log 2>&1
export TOFR_B200_LIB=$V/libtofr_b200_phist.so
bash tools/gpu_run.sh r02p kprof:c4p:k_hist_plain:1:25 > /dev/null 2>&1
mv $O/kprof_c4p_k_hist_plain.txt $O/kprof_c4p_k_hist_plain_phist.txt; mv $O/kprof.log $O/kprof_phist.log
unset TOFR_B200_LIB
