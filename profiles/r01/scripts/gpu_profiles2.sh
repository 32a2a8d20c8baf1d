#!/bin/bash
# Profile artefacts for profiles/<tag>/: GPU suite + smoke, bench lines of every
# workload (+ the reference arm), ncu launch lists, and ncu --set full captures
# of each workload's dominant kernels over one steady-state frame's launches.
#   bash tools/gpu_profiles2.sh <tag>
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu.txt
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for wl in c3w c3d c5 c1 c2p c2r c4p; do
  timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 900 python bench.py --workload c4r --steps 10 --warmup 3 > $O/bench_c4r.json 2> $O/bench_c4r.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
# launch lists (serialised, cold-ish caches: shares, not absolutes)
for wl in c3 c3w c2r; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$wl.csv \
      python bench.py --workload $wl --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  python tools/ncu_summary.py launches $O/launches_$wl.csv > $O/launches_${wl}_summary.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4r.csv \
    python bench.py --workload c4r --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py launches $O/launches_c4r.csv > $O/launches_c4r_summary.txt 2>&1
# full captures: <workload> <file tag = library kernel name> <ncu regex> <skip> <count>
# (reports are ~5 MB per launch and gpurun brings back <= 64 MiB: each one is
# summarised on the box -- metrics, DRAM traffic, hot source lines -- then dropped)
cap() {
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$3" -s $4 -c $5 -o $O/full_$1_$2 \
      python bench.py --workload $1 --steps 2 --warmup 4 --no-cpu-baseline > $O/ncu_full_$1_$2.log 2>&1
  python tools/ncu_summary.py full $O/full_$1_$2.ncu-rep > $O/full_$1_$2.txt 2>&1
  python tools/traffic_json.py --out $O/traffic.json $O/full_$1_$2.ncu-rep >> $O/traffic.log 2>&1
  ncu -i $O/full_$1_$2.ncu-rep --page source --print-source cuda,sass --csv --launch-count 1 > /tmp/src.csv 2>/dev/null
  python tools/ncu_lines.py /tmp/src.csv 30 > $O/lines_$1_$2.txt 2>&1
  rm -f $O/full_$1_$2.ncu-rep
}
cap c3 k_shift_solve '^k_shift_solve' 16 4
cap c3 k_trace_gated '^k_trace' 4 1
cap c3w k_shift_solve '^k_shift_solve' 16 4
cap c3w k_shift_finish '^k_shift_finish' 16 4
cap c3w k_trace_gated '^k_trace' 4 1
cap c2r k_shift_finish '^k_shift_finish' 8 2
cap c2r k_temporal_apply '^k_temporal_apply' 8 2
cap c2r k_temporal_prep '^k_temporal_prep' 8 2
cap c4p k_hist_plain '^k_hist_plain' 4 1
ls $O
# one raw report kept for inspection (one steady-state launch of the headline's dominant kernel)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_shift_solve' -s 17 -c 1 \
    -o $O/keep_c3_k_shift_solve python bench.py --workload c3 --steps 2 --warmup 4 --no-cpu-baseline > /dev/null 2>&1
du -sh $O
