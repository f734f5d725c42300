cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py -q -rf --timeout 600 > gpurun_out/pytest_rgp.log 2>&1; echo "rc=$?"; tail -25 gpurun_out/pytest_rgp.log
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_boundary.py -q -x -rf --timeout 600 2>&1 | tail -3
