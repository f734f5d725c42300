cd $GRAFT_REPO_ROOT
timeout 300 python tools/pcie_probe.py 2>&1 | tail -1
timeout 600 python tools/probe_e2e.py 2>&1 | tail -1
