cd $GRAFT_REPO_ROOT
QSIM_PLAN_LOG=1 timeout 300 python tools/probe_cfg4.py 24 > gpurun_out/cfg4_24.json 2> gpurun_out/cfg4_24.plan; echo rc=$?
QSIM_PLAN_LOG=1 timeout 600 python tools/probe_cfg4.py 32 > gpurun_out/cfg4_32.json 2> gpurun_out/cfg4_32.plan; echo rc=$?
tail -c 1500 gpurun_out/cfg4_32.json; grep -c "qsim plan" gpurun_out/cfg4_32.plan
