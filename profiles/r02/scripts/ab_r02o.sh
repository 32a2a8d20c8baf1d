V=paper_2605_11536_b200/_native/variants
for lib in default noshare; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  python tools/band_kernels.py c3 8 2 > gpurun_out/r02o/bk82_$lib.log 2>&1
  python tools/band_kernels.py c3 8 7 > gpurun_out/r02o/bk87_$lib.log 2>&1
  python bench.py --workload c3 --steps 20 --warmup 25 --no-cpu-baseline > gpurun_out/r02o/c3_$lib.json 2>/dev/null
  python bench.py --workload nlos --steps 20 --warmup 25 --no-cpu-baseline > gpurun_out/r02o/nlos_$lib.json 2>/dev/null
  python bench.py --workload c1 --steps 20 --warmup 25 --no-cpu-baseline > gpurun_out/r02o/c1_$lib.json 2>/dev/null
done
unset TOFR_B200_LIB
export TOFR_B200_LIB=$V/libtofr_b200_sprof.so; python tools/solve_profile.py c3 8 2 > gpurun_out/r02o/sp82_share.log 2>&1
export TOFR_B200_LIB=$V/libtofr_b200_sprof_noshare.so; python tools/solve_profile.py c3 8 7 > gpurun_out/r02o/sp87_noshare.log 2>&1
export TOFR_B200_LIB=$V/libtofr_b200_sprof.so; python tools/solve_profile.py c3 8 7 > gpurun_out/r02o/sp87_share.log 2>&1
unset TOFR_B200_LIB
python tools/band_probe2.py c3 8 > gpurun_out/r02o/probe_c3_8.log 2>&1
for i in 1 2; do
  for lib in default phist; do
    if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
    python bench.py --workload c4p --steps 20 --warmup 25 --no-cpu-baseline > gpurun_out/r02o/c4p_${lib}_$i.json 2>/dev/null
    python bench.py --workload c2p --steps 20 --warmup 25 --no-cpu-baseline > gpurun_out/r02o/c2p_${lib}_$i.json 2>/dev/null
  done
done
