# solve CTAs per SM (room for the side stream's next-frame init)
O=gpurun_out/r02au; mkdir -p $O
for c in 0 3 2; do
  for wl in c3 c3w c1; do
    TOFR_SOLVE_CTAS=$c python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/${wl}_$c.json 2>/dev/null
  done
done
for f in $O/*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['value'],1),round(d['e2e']['value'],1))"; done > $O/summary.txt
