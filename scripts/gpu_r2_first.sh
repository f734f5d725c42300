set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_fullsize.py -m gpu -q -rf -s --timeout 1200 > gpurun_out/pytest_new.log 2>&1; echo "new rc=$?"
tail -40 gpurun_out/pytest_new.log
timeout 1500 python -m pytest tests -m gpu -q -rf -x --timeout 600 --deselect tests/test_gpu_fullsize.py --deselect tests/test_gpu_boundary.py > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -20 gpurun_out/pytest_gpu.log
