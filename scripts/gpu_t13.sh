cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_races.py -q --timeout 600 -rf 2>&1 | tail -8
