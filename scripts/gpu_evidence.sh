# round evidence: full bench line, per-config timings, per-gate table, launch list, ncu of the dominant kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_full.log | cut -c1-3000
timeout 1200 python tools/bench_configs.py 0 1 2 3 3n 4 f1 f4 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
cut -c1-300 gpurun_out/configs.jsonl; tail -3 gpurun_out/configs.err
REPS=5 timeout 900 python tools/bench_gates.py 28 30 32 > gpurun_out/gates.jsonl 2> gpurun_out/gates.err; echo "gates rc=$?"
CMD="python bench.py --profile-only --steps 2 --warmup 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
CMD1="python bench.py --profile-only --steps 1 --warmup 1"
timeout 300 $CMD1 > gpurun_out/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_qft_tma -c 4 -o gpurun_out/prof_qft $CMD1 > gpurun_out/ncu_qft.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_qft.log
ncu -i gpurun_out/prof_qft.ncu-rep --page details > gpurun_out/prof_qft_details.txt 2>&1
ncu -i gpurun_out/prof_qft.ncu-rep --page raw --csv > gpurun_out/prof_qft_raw.csv 2>&1
rm -f gpurun_out/prof_qft.ncu-rep
