cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "hadamard or had" 2>&1 | tail -2
for n in 26 28 29 30; do echo "$(timeout 300 python tools/probe_qft3.py $n had 2>&1 | tail -1 | cut -c1-260)"; done
