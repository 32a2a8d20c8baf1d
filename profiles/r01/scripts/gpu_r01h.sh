#!/bin/bash
# Re-entry measurement pass: full GPU suite, smoke, bench lines for every workload,
# launch list of the headline bench, one full ncu capture of the spatial kernels.
O=gpurun_out/r01h
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > $O/bench_c3.json 2> $O/bench_c3.err
for wl in c3w c5 c1 c2p c2r c4p; do
  timeout 400 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_spatial_fwd$|k_spatial_merge|k_temporal|k_init_gated' \
    -s 8 -c 5 -o $O/prof_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_full.log 2>&1
ls -la $O
