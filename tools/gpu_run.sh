#!/bin/bash
# Parameterised GPU-box run: bash tools/gpu_run.sh <tag> <steps...>
#   steps: tests | smoke | bench:<wl>[:<extra args>] | ref | launches:<wl> | full:<wl>:<kernel regex>:<skip>:<count>
TAG=${1:-run}; shift
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" >> $O/gpu.txt; free -g >> $O/gpu.txt
for s in "$@"; do
  IFS=: read -r kind a b c d <<< "$s"
  case $kind in
    tests) timeout ${a:-1800} python -m pytest tests -m gpu -q -x ${b:+-k "$b"} > $O/pytest_gpu${b:+_$b}.log 2>&1; tail -3 $O/pytest_gpu${b:+_$b}.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log ;;
    bench) timeout 900 python bench.py --workload $a --steps ${c:-20} --warmup ${d:-25} ${b:+$b} > $O/bench_$a.json 2> $O/bench_$a.err; tail -c 600 $O/bench_$a.json ;;
    ref) timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$a.csv \
        python bench.py --workload $a --steps 2 --warmup ${b:-25} --no-cpu-baseline > /dev/null 2>&1
      python tools/ncu_summary.py launches $O/launches_$a.csv > $O/launches_${a}_summary.txt 2>&1 ;;
    full) timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$b" -s $c -c $d -o $O/full_${a}_$(echo $b|tr -dc a-z_) \
        python bench.py --workload $a --steps 2 --warmup 25 --no-cpu-baseline > $O/ncu_full_$a.log 2>&1
      f=$O/full_${a}_$(echo $b|tr -dc a-z_)
      python tools/ncu_summary.py full $f.ncu-rep > $f.txt 2>&1
      ncu -i $f.ncu-rep --page source --print-source cuda,sass --csv --launch-count 1 > /tmp/src.csv 2>/dev/null
      python tools/ncu_lines.py /tmp/src.csv 30 > ${f/full_/lines_}.txt 2>&1
      rm -f $f.ncu-rep ;;
    kprof) # kprof:<wl>:<kernel>:<launches per frame>:<warm> -> profiles-ready kernel_profile.json entry
      W=${d:-25}; L=${c:-1}; f=$O/kprof_${a}_$b; K=$b
      case $b in k_trace_*) K=k_trace ;; esac   # the library names k_trace's instantiations per sink
      timeout 1800 ncu --set full --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum \
          --clock-control none --import-source on -k regex:"^$K(<|\\(|$)" -s $((W * L)) -c $L -o $f \
          python bench.py --workload $a --steps 1 --warmup $W --no-cpu-baseline > $f.json 2> $f.err
      python tools/kernel_profile.py --out $O/kernel_profile.json --wl $a --kernel $b --bench $f.json $f.ncu-rep >> $O/kprof.log 2>&1
      python tools/ncu_summary.py full $f.ncu-rep > $f.txt 2>&1
      ncu -i $f.ncu-rep --page source --print-source cuda,sass --csv --launch-count 1 > /tmp/src.csv 2>/dev/null
      python tools/ncu_lines.py /tmp/src.csv 30 > ${f/kprof_/lines_}.txt 2>&1
      rm -f $f.ncu-rep; tail -1 $O/kprof.log ;;
    cmd) eval "$a" > $O/cmd_${b:-x}.log 2>&1; tail -5 $O/cmd_${b:-x}.log ;;
  esac
done
ls $O
