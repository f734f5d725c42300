cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py -q -x --timeout 600 2>&1 | tail -1
for n in 28 29; do
  for r in 1 2; do echo "$(timeout 300 python tools/probe_qft3.py $n qft 2>&1 | tail -1 | cut -c1-250)"; done
done
