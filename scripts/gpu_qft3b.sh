cd $GRAFT_REPO_ROOT
for B in default 10,9,9 9,10,9; do
   if [ "$B" = default ]; then unset QSIM_QFT_BLOCKS; else export QSIM_QFT_BLOCKS=$B; fi
   timeout 120 python tools/probe_qft3.py 28 had 2>&1 | tail -1
done | tee gpurun_out/qft3b.jsonl
