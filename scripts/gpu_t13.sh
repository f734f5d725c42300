cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py -q -x --timeout 600 -k "falls_back or free" -rA 2>&1 | grep -v "^PASSED" | tail -6
