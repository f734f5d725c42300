# end-of-round check: the driver's three steps (GPU tests, smoke, default bench)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/final_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/final_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['steps'], d['warmup'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'])"
