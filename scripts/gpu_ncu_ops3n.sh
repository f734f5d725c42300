# ncu of the heavy noisy-QFT gate-list pass of configs[3] sigma = 1e-3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/run_cfg.py 3n"
timeout 300 $CMD > gpurun_out/plain_3n.log 2>&1
echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ops_pass -s 2 -c 1 -o gpurun_out/prof_3n $CMD > gpurun_out/ncu_3n.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_3n.log
ncu -i gpurun_out/prof_3n.ncu-rep --page raw --csv > gpurun_out/prof_3n_raw.csv 2>&1
ncu -i gpurun_out/prof_3n.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_3n_sass.csv 2>&1
