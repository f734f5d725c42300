cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_group.py tests/test_gpu_boundary.py tests/test_gpu_next.py -q -x -rf --timeout 600 2>&1 | tail -3
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel'], d['nvlink'], d['kernels'].keys())"
