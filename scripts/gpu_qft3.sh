cd $GRAFT_REPO_ROOT
for B in default 10,9,9 9,10,9 9,9,10 10,10,8; do
 for P in -1 256 128; do
  for G in 0 2; do
   if [ "$B" = default ]; then unset QSIM_QFT_BLOCKS; else export QSIM_QFT_BLOCKS=$B; fi
   if [ "$P" = -1 ]; then unset QSIM_L2PROM; else export QSIM_L2PROM=$P; fi
   QSIM_TILE_GROUP=$G timeout 120 python tools/probe_qft3.py 28 2>&1 | tail -1
  done
 done
done | tee gpurun_out/qft3.jsonl
