# gate-list pass change: parity + configs timings with and without it, plan log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_configs.py ${CFGS:-4 3n 0} > gpurun_out/cfg_new.jsonl 2> gpurun_out/cfg_new.err; echo "cfg rc=$?"
tail -3 gpurun_out/cfg_new.err
env ${OFFENV:-QSIM_NO_DENSE4}=1 timeout 600 python tools/bench_configs.py ${CFGS:-4 3n 0} > gpurun_out/cfg_old.jsonl 2> gpurun_out/cfg_old.err; echo "cfg old rc=$?"
QSIM_PLAN_LOG=1 timeout 300 python tools/run_cfg.py 4m > gpurun_out/plan_4m.log 2>&1
