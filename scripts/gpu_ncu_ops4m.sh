# ncu of a heavy gate-list pass of configs[4] at n = 30 (the n = 32 pattern, a quarter of the state)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/run_cfg.py 4m"
QSIM_PLAN_LOG=1 timeout 300 $CMD > gpurun_out/plain_4m.log 2>&1
echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_ops_pass -s 3 -c 1 -o gpurun_out/prof_4m $CMD > gpurun_out/ncu_4m.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_4m.log
ncu -i gpurun_out/prof_4m.ncu-rep --page raw --csv > gpurun_out/prof_4m_raw.csv 2>&1
ncu -i gpurun_out/prof_4m.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_4m_sass.csv 2>&1
