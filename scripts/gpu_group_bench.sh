cd $GRAFT_REPO_ROOT
for g in 2 4; do
timeout 900 python bench.py --gpus $g --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g$g.log 2>&1; echo "g$g rc=$?"
tail -1 gpurun_out/bench_g$g.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config'].get('parallelism'), d['roofline']['kernel'], round(d['roofline']['frac'],3), json.dumps(d.get('nvlink'))[:300], d.get('kernels',{}).keys())"
done
