cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_parity.py -k "qft or hadamard or cfg2" -q -x -rf --timeout 600 > gpurun_out/pytest_qft13.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_qft13.log
for B in default 9,10,9; do
   if [ "$B" = default ]; then unset QSIM_QFT_BLOCKS; else export QSIM_QFT_BLOCKS=$B; fi
   timeout 120 python tools/probe_qft3.py 28 2>&1 | tail -1
done | tee gpurun_out/qft13.jsonl
unset QSIM_QFT_BLOCKS
for n in 26 27 29 30; do timeout 120 python tools/probe_qft3.py $n 2>&1 | tail -1; done | tee -a gpurun_out/qft13.jsonl
