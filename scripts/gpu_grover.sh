cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_races.py tests/test_gpu_boundary.py -k "grover or cfg1 or diffusion" -q -rf --timeout 600 2>&1 | tail -3
for v in 0 1; do
if [ $v = 1 ]; then export QSIM_GROVER_REDUCE=1; else unset QSIM_GROVER_REDUCE; fi
timeout 300 python tools/bench_configs.py 1 2>&1 | tail -1 | cut -c1-400
done
