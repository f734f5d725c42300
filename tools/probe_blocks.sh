# QFT block partitions (experiment; QSIM_QFT_BLOCKS), n from $N (default 28)
cd $GRAFT_REPO_ROOT
N=${N:-28}
for b in $BLOCKS; do
  for i in 1 2; do
    QSIM_QFT_BLOCKS=$b timeout 300 python bench.py --n $N --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$N', '$b', round(d['ms_per_step'],4), round(d['roofline']['frac'],4))"
  done
done
