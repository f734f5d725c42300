cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shor.py -m gpu -q -x --timeout 900 -k "qft or cfg3 or shor or order or free or had" 2>&1 | tail -2
for v in 0 1; do
if [ $v = 1 ]; then export QSIM_NO_QFLEX=1; else unset QSIM_NO_QFLEX; fi
timeout 300 python tools/bench_configs.py 3 2>&1 | tail -1 | cut -c1-330
done
unset QSIM_NO_QFLEX
for n in 28 29; do echo "$(timeout 300 python tools/probe_qft3.py $n qft 2>&1 | tail -1 | cut -c1-250)"; done
