# ncu of the fused gate-list kernel on configs[4] at n = 26 (+ the planner's pass log)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/run_cfg.py 4s"
QSIM_PLAN_LOG=1 timeout 300 $CMD > gpurun_out/plain_ops.log 2>&1
echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ops_pass -s 8 -c 1 -o gpurun_out/prof_ops $CMD > gpurun_out/ncu_ops.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_ops.log
ncu -i gpurun_out/prof_ops.ncu-rep --page raw --csv > gpurun_out/prof_ops_raw.csv 2>&1
ncu -i gpurun_out/prof_ops.ncu-rep --page details --csv > gpurun_out/prof_ops_details.csv 2>&1
ncu -i gpurun_out/prof_ops.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ops_sass.csv 2>&1
