O=gpurun_out/ab_pipe_tr; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -1 $O/pytest_gpu.log | tee -a $O/summary.txt
for wl in t1080b64 c2r t1080 t1080b64; do for dp in 3 2; do
  TOFR_PIPE_DEPTH=$dp timeout 900 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$dp.json 2> $O/$wl.$dp.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['value'],2), round(d['e2e']['value'],2), d.get('reservoir_pool'))" $O/$wl.$dp.json "$wl depth=$dp" | tee -a $O/summary.txt
done; done
