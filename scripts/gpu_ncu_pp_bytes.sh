cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/run_cfg.py 4m > /dev/null 2>&1
QSIM_OPS_PP_MAX=100 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_ops_pp -c 3 --csv python tools/run_cfg.py 4m > gpurun_out/pp_bytes.csv 2>/dev/null
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_ops_pp -c 2 --csv python tools/run_cfg.py 3n > gpurun_out/pp_bytes3n.csv 2>/dev/null
grep -h "k_ops_pp" gpurun_out/pp_bytes.csv gpurun_out/pp_bytes3n.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -20
