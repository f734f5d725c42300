cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py -q -x --timeout 600 -k "free_layouts" 2>&1 | tail -3
