O=gpurun_out/v4; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log | tee -a $O/summary.txt
for wl in c1 c3 c3w c2r t1080b64 nlos; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 900 python bench.py --workload c4r --steps 6 --warmup 25 --no-cpu-baseline > $O/bench_c4r.json 2> $O/bench_c4r.err
