#!/bin/bash
# variant sweep: register caps (TOFR_REUSE_MINB) after moving traversal/shift out of line
mkdir -p gpurun_out/r01b
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01b/pytest_gpu.log 2>&1
for v in main m3 m4; do
  if [ $v = main ]; then unset TOFR_B200_LIB; else export TOFR_B200_LIB=paper_2605_11536_b200/_native/variants/libtofr_b200_$v.so; fi
  for wl in c3 c3w; do
    timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01b/bench_${v}_${wl}.json 2>&1
  done
done
