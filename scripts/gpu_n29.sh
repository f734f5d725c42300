cd $GRAFT_REPO_ROOT
for B in 10,10,9 10,9,10 9,10,10; do QSIM_QFT_BLOCKS=$B timeout 120 python tools/probe_qft3.py 29 2>&1 | tail -1; done
for B in 10,10,10 8,8,7,7; do QSIM_QFT_BLOCKS=$B timeout 120 python tools/probe_qft3.py 30 2>&1 | tail -1; done
for B in 10,10,10,3 8,8,8,7 9,8,8,8; do QSIM_QFT_BLOCKS=$B timeout 120 python tools/probe_qft3.py 31 2>&1 | tail -1; done
