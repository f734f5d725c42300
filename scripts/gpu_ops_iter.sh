# quick iteration on the gate-list kernel: parity suite + noisy config timings + pass log
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/bench_configs.py ${CFGS:-4 3n 4s} > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg rc=$?"
tail -3 gpurun_out/cfg4.err; cut -c1-600 gpurun_out/cfg4.jsonl
QSIM_PLAN_LOG=1 timeout 300 python tools/run_cfg.py 4s > gpurun_out/plan_4s.log 2>&1
