cd $GRAFT_REPO_ROOT
python tools/bench_configs.py 1 > gpurun_out/plain_grover.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_grover_regs -s 1 -c 1 -o gpurun_out/r2_prof_grover python tools/bench_configs.py 1 > gpurun_out/ncu_grover.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/r2_prof_grover.ncu-rep --print-summary none > gpurun_out/r2_ncu_k_grover_regs.txt 2>&1; wc -l gpurun_out/r2_ncu_k_grover_regs.txt
