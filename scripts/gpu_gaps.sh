cd $GRAFT_REPO_ROOT
timeout 300 python tools/probe_gaps.py 28 2>&1 | tail -2
timeout 300 python tools/probe_gaps.py 26 2>&1 | tail -2
