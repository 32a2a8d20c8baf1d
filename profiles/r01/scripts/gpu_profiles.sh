#!/bin/bash
# Profile artefacts for profiles/: bench lines, launch lists, and one ncu --set full
# capture of each workload's dominant kernel (dram traffic per launch -> traffic.json).
#   bash tools/gpu_profiles.sh <tag>
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for wl in c3w c5 c1 c2p c2r c4p; do
  timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
# launch lists (serialised, cold-ish caches: shares, not absolutes)
for wl in c3 c3w c2r; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$wl.csv \
      python bench.py --workload $wl --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_summary.py launches $O/launches_$wl.csv > $O/launches_${wl}_summary.txt
done
# full captures of the dominant kernels (steady-state frame 3: skip the earlier launches)
cap() {  # workload kernel skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$2" -s $3 -c 1 -o $O/full_$1_$2 \
      python bench.py --workload $1 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full_$1_$2.log 2>&1
  python tools/ncu_summary.py full $O/full_$1_$2.ncu-rep > $O/full_$1_$2.txt 2>&1
}
cap c3 k_shift_solve 15
cap c3 k_trace 3
cap c3w k_trace 3
cap c3w k_shift_solve 15
cap c3w k_shift_finish 15
cap c2r k_temporal_prep 3
cap c2r k_temporal_apply 3
cap c4p k_hist_plain 3
ls $O
