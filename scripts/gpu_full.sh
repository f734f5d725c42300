cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 -rf 2>&1 | tail -40 > gpurun_out/full_tests.log
cat gpurun_out/full_tests.log
