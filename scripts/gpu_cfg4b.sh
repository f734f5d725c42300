cd $GRAFT_REPO_ROOT
for i in 1 2; do timeout 600 python tools/probe_cfg4.py 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['wall_s'], d['kernel_ms'])"; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "cfg4 or cfg0 or random or ctrl or batch or mixed" --timeout 600 2>&1 | tail -2
