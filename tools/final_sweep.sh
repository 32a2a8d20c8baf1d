# Round-end evidence: GPU suite (incl. compute-sanitizer), smoke, ncu kernel
# profiles of the kernels changed last, then every bench line with those
# profiles merged in, the reference arm and launch lists.
#   bash tools/final_sweep.sh <tag>
TAG=${1:-final}; O=gpurun_out/$TAG; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --timeout 1800 > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
bash tools/gpu_run.sh $TAG kprof:c3:k_shift_solve:4:25 kprof:c2r:k_shift_finish:4:25 kprof:t1080b64:k_shift_finish:8:25 kprof:t1080b64:k_shift_solve:8:25 kprof:t1080b64:k_temporal_apply:8:25 > /dev/null 2>&1
python - <<PY
import json
p='profiles/kernel_profile.json'; d=json.load(open(p)); n=json.load(open('$O/kernel_profile.json'))
for k,v in n.items(): v['source'] += ' [$TAG]'; d[k]=v
json.dump(d, open(p,'w'), indent=1, sort_keys=True); json.dump(d, open('$O/kernel_profile_merged.json','w'), indent=1, sort_keys=True)
PY
timeout 900 python bench.py --steps 20 --warmup 25 > $O/bench_c3.json 2> $O/bench_c3.err
for wl in c3d c3w c3w_shrink c1 c2p c2r c2r_bin c4p t1080b64 t1080 nlos nlos_scan mesh mesh_anim; do
  timeout 900 python bench.py --workload $wl --steps 20 --warmup 25 --no-cpu-baseline > $O/bench_$wl.json 2> $O/bench_$wl.err
done
timeout 900 python bench.py --workload c5 --steps 120 --warmup 25 --no-cpu-baseline > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1500 python bench.py --workload c4r --steps 10 --warmup 25 --no-cpu-baseline > $O/bench_c4r.json 2> $O/bench_c4r.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
bash tools/gpu_run.sh $TAG launches:c3 launches:c2r > /dev/null 2>&1
ls $O
