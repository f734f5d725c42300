cd $GRAFT_REPO_ROOT
python tools/probe_cfg4.py 32 > gpurun_out/plain_ops.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ops_pp -s 3 -c 1 -o gpurun_out/r2_prof_ops python tools/probe_cfg4.py 32 > gpurun_out/ncu_ops.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2_prof_ops.ncu-rep --print-summary none > gpurun_out/r2_ncu_k_ops_pp.txt 2>&1; wc -l gpurun_out/r2_ncu_k_ops_pp.txt
