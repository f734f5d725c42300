cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -rf --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu.log
python tools/probe_lowgates.py 2>&1 | tee gpurun_out/lowgates_default.jsonl
timeout 600 python tools/probe_cfg4.py 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['wall_s'], d['kernel_ms'])"
