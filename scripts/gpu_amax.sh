cd $GRAFT_REPO_ROOT
for A in 10 9 8 7; do
  QSIM_QFT_AMAX=$A timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_a$A.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_a$A.log").read().strip().splitlines()[-1])
print("amax=$A", "ms=%.3f"%d["ms_per_step"], "passes=%.1f"%d["roofline"]["launches_per_step"], "pass_ms=%.3f"%d["roofline"]["ms_per_launch"], "GB/s=%.0f"%d["roofline"]["achieved"])
PY
done
