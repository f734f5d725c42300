cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_qft13.py tests/test_gpu_fullsize.py -k "qft13 or hadamard13 or fft13 or cfg2 or cfg4" -q -x -rf --timeout 600 > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pdl.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl', d['ms_per_step'], d['roofline']['ms_per_launch'], d['e2e']['ms_per_step'])"
QSIM_NO_PDL=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nopdl', d['ms_per_step'], d['roofline']['ms_per_launch'], d['e2e']['ms_per_step'])"
done
