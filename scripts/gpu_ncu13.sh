cd $GRAFT_REPO_ROOT
python tools/probe_qft3.py 28 > gpurun_out/plain13.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qft13 -s 6 -c 3 -o gpurun_out/prof13 python tools/probe_qft3.py 28 > gpurun_out/ncu13.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu13.log
