cd $GRAFT_REPO_ROOT
python tools/probe_cfg4.py 28 4 > gpurun_out/plain_ops.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ops_pp -s 4 -c 2 -o gpurun_out/prof_ops python tools/probe_cfg4.py 28 4 > gpurun_out/ncu_ops.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_ops.log
