cd $GRAFT_REPO_ROOT
UNFUSED=1 python tools/probe_lowgates.py > gpurun_out/lowgates_unf.jsonl 2>&1 && cat gpurun_out/lowgates_unf.jsonl && \
UNFUSED=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lowgates_unf_ncu.csv python tools/probe_lowgates.py > /dev/null 2>&1
echo rc=$?
