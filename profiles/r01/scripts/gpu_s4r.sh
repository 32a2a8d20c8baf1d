O=gpurun_out/${TAG:-s4r}; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
for wl in c3 c3w c1; do
  timeout 400 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
  python -c "import json; d=json.load(open('$O/bench_$wl.json')); print('$wl', round(d['value'],2), d['stage_ms'], 'e2e', round(d['e2e']['value'],2))" || tail -5 $O/bench_$wl.err
done
timeout 600 python bench.py --workload c4r --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c4r.json 2> $O/bench_c4r.err
python -c "import json; d=json.load(open('$O/bench_c4r.json')); print('c4r', round(d['value'],3), d['stage_ms'], 'e2e', round(d['e2e']['value'],3), list(d['kernel_ms_per_step'].items())[:6])" || tail -5 $O/bench_c4r.err
