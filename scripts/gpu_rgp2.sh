cd $GRAFT_REPO_ROOT
for g in 2 4; do
for v in 0 1; do
if [ $v = 1 ]; then export QSIM_NO_RANK_GROUP_PASS=1; else unset QSIM_NO_RANK_GROUP_PASS; fi
timeout 600 python bench.py --gpus $g --steps 10 --warmup 3 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpus', $g, 'no_rgp', $v, round(d['ms_per_step'],3), d['kernels'].keys(), d['nvlink'] and round(d['nvlink']['ms_per_step'],3))"
done; done
