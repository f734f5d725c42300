cd $GRAFT_REPO_ROOT
timeout 600 python tools/probe_sustained.py 2>&1 | tail -30
