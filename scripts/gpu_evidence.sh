# round evidence: full bench line, per-config timings, launch list, ncu of the dominant kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log | cut -c1-3000
timeout 900 python tools/bench_configs.py 0 1 2 3 3n 4s > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
cat gpurun_out/configs.jsonl | cut -c1-600; tail -3 gpurun_out/configs.err
CMD="python bench.py --profile-only --steps 2 --warmup 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD1="python bench.py --profile-only --steps 1 --warmup 1"
timeout 300 $CMD1 > gpurun_out/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft_tma -c 4 -o gpurun_out/prof_qft $CMD1 > gpurun_out/ncu_qft.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_qft.log
