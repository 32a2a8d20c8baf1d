O=gpurun_out/nscan; mkdir -p $O
for dp in 3 2 3; do TOFR_PIPE_DEPTH=$dp timeout 600 python bench.py --workload nlos_scan --steps 20 --warmup 25 --no-cpu-baseline > $O/ns.$dp.json 2> $O/ns.$dp.err; python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('nlos_scan depth', sys.argv[2], round(d['value'],2), round(d['e2e']['value'],2))" $O/ns.$dp.json $dp | tee -a $O/summary.txt; done
bash profiles/r02/scripts/ab_take.sh
