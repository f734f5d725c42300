cd $GRAFT_REPO_ROOT
for n in 24 26 27 28 29 30 31; do timeout 120 python tools/probe_qft3.py $n 2>&1 | tail -1; done > gpurun_out/r2_qft_sizes.jsonl
for n in 28 30; do timeout 120 python tools/probe_qft3.py $n had 2>&1 | tail -1; done >> gpurun_out/r2_qft_sizes.jsonl
cat gpurun_out/r2_qft_sizes.jsonl
python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_l.log 2>&1
echo "ncu rc=$?"
