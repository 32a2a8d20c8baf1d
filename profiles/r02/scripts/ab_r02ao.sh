O=gpurun_out/r02ao; mkdir -p $O
V=paper_2605_11536_b200/_native/variants
for lib in default esc2 esc3; do
  if [ $lib = default ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=$V/libtofr_b200_$lib.so; fi
  python tools/band_probe2.py c3w 8 > $O/bp_c3w_$lib.log 2>&1
  python tools/band_probe2.py c3 8 > $O/bp_c3_$lib.log 2>&1
  python bench.py --workload c3w --steps 20 --warmup 25 --no-cpu-baseline > $O/c3w_$lib.json 2>/dev/null
done
