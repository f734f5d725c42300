# per-config table (tools/bench_configs.py) + H_n / QFT pass probes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python tools/bench_configs.py 0 1 2 3 3n 4 > gpurun_out/r2_configs.jsonl 2> gpurun_out/r2_configs.err; echo "configs rc=$?"
for n in 28 30; do for op in qft had; do timeout 300 python tools/probe_qft3.py $n $op 2>&1 | tail -1; done; done > gpurun_out/r2_probe.jsonl
cat gpurun_out/r2_probe.jsonl | cut -c1-250
