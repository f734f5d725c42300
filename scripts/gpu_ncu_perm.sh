# ncu of the MODEXP permutation of configs[3] (sigma = 0)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/run_cfg.py 3"
timeout 300 $CMD > gpurun_out/plain_3.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_perm -c 1 -o gpurun_out/prof_perm $CMD > gpurun_out/ncu_perm.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_perm.log
ncu -i gpurun_out/prof_perm.ncu-rep --page raw --csv > gpurun_out/prof_perm_raw.csv 2>&1
ncu -i gpurun_out/prof_perm.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_perm_src.csv 2>&1
