cd $GRAFT_REPO_ROOT
for oop in 0 1; do
  if [ $oop = 1 ]; then export QSIM_Q13_OOP=1; else unset QSIM_Q13_OOP; fi
  for b in default 9,10,9; do
    if [ $b = default ]; then unset QSIM_QFT_BLOCKS; else export QSIM_QFT_BLOCKS=$b; fi
    for r in 1 2; do
    echo "oop=$oop $(timeout 300 python tools/probe_qft3.py 28 qft 2>&1 | tail -1 | cut -c1-250)"
    done
  done
done
