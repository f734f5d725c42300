cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_races.py -q -rf --timeout 600 > gpurun_out/pytest_races.log 2>&1; echo "races rc=$?"; tail -3 gpurun_out/pytest_races.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks_r2.csv &
SMI=$!
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.log 2>&1; echo "bench rc=$?"
kill $SMI
tail -c 1500 gpurun_out/bench_r2.log
python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_qft13 -s 9 -c 3 -o gpurun_out/r2_prof_qft13 python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_r2.log 2>&1
echo "ncu rc=$?"
