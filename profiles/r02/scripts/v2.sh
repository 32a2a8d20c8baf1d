O=gpurun_out/v2; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
val() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(round(d['value'],2), round(d['e2e']['value'],2))" $1; }
for wl in mesh c3 c3d; do for dp in 3 2; do
  TOFR_PIPE_DEPTH=$dp timeout 600 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/$wl.$dp.json 2> $O/$wl.$dp.err
  echo "$wl depth=$dp $(val $O/$wl.$dp.json)" | tee -a $O/summary.txt
done; done
