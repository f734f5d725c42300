# round-2 evidence: smoke, per-config table, the driver's bench line, configs[4] line, reference arm, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python tools/bench_configs.py 0 1 2 3 3n 4 > gpurun_out/r2_configs.jsonl 2> gpurun_out/r2_configs.err; echo "configs rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench.log | cut -c1-300
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/r2_bench_cfg4.log 2>&1; echo "cfg4 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r2_bench_ref.log | cut -c1-300
python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/plain_prof.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --profile-only > gpurun_out/ncu_launch.log 2>&1
echo "ncu rc=$?"
