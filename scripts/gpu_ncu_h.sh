cd $GRAFT_REPO_ROOT
python tools/probe_qft3.py 28 had > gpurun_out/plain_h.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qft13 -s 6 -c 3 -o gpurun_out/r2_prof_h python tools/probe_qft3.py 28 had > gpurun_out/ncu_h.log 2>&1
echo "ncu rc=$?"
