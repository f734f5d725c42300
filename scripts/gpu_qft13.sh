cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py -q -x -rf --timeout 600 > gpurun_out/pytest_qft13.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_qft13.log
for B in default 10,9,9 9,10,9 10,10,8; do
   if [ "$B" = default ]; then unset QSIM_QFT_BLOCKS; else export QSIM_QFT_BLOCKS=$B; fi
   timeout 120 python tools/probe_qft3.py 28 2>&1 | tail -1
   timeout 120 python tools/probe_qft3.py 28 had 2>&1 | tail -1
done | tee gpurun_out/qft13.jsonl
unset QSIM_QFT_BLOCKS
for n in 26 27 29 30; do timeout 120 python tools/probe_qft3.py $n 2>&1 | tail -1; done | tee -a gpurun_out/qft13.jsonl
QSIM_NO_QFT13=1 timeout 120 python tools/probe_qft3.py 28 2>&1 | tail -1
