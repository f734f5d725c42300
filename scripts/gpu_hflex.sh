# H with free intermediate layouts (R42): parity, then pass times with / without (QSIM_NO_HFLEX)
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -k "hadamard or Hadamard or had or cfg3 or cfg1 or grover or shor or ht_ or batch or group" 2>&1 | tail -3
for v in 0 1; do
  if [ $v = 1 ]; then export QSIM_NO_HFLEX=1; else unset QSIM_NO_HFLEX; fi
  for n in 24 26 28 29 30; do echo "nohflex=$v $(timeout 300 python tools/probe_qft3.py $n had 2>&1 | tail -1 | cut -c1-260)"; done
  timeout 300 python tools/bench_configs.py 3 2>&1 | tail -1 | cut -c1-330
done
