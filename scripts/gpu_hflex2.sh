cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 -k "hadamard or had or free" 2>&1 | tail -2
for v in 0 1; do
if [ $v = 1 ]; then export QSIM_NO_ST256=1; else unset QSIM_NO_ST256; fi
for n in 26 28 29 30; do echo "nost256=$v $(timeout 300 python tools/probe_qft3.py $n had 2>&1 | tail -1 | cut -c1-260)"; done
echo "nost256=$v $(timeout 300 python tools/probe_qft3.py 28 qft 2>&1 | tail -1 | cut -c1-260)"
done
