cd $GRAFT_REPO_ROOT
for i in 1 2; do
QSIM_LIB=$GRAFT_REPO_ROOT/paper_quant_ph_0201042_b200/libqsim_a.so timeout 600 python tools/probe_cfg4.py 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['wall_s'], d['kernel_ms'])"
timeout 600 python tools/probe_cfg4.py 32 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['wall_s'], d['kernel_ms'])"
done
