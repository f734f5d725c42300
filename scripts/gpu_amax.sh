cd $GRAFT_REPO_ROOT
for A in 10 9 7 6 5; do
  QSIM_QFT_AMAX=$A timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_a$A.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_a$A.log").read().strip().splitlines()[-1])
print("amax=$A", "ms=%.3f"%d["ms_per_step"], d["roofline"]["kernel"], "passes", d["step_launches_ms"])
PY
done
