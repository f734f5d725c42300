cd $GRAFT_REPO_ROOT
CMD="python tools/run_cfg.py 4s"
timeout 300 $CMD > gpurun_out/plain_ops.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ops -c 3 -o gpurun_out/prof_ops $CMD > gpurun_out/ncu_ops.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_ops.log
