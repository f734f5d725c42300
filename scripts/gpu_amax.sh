cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "qft or hadamard or cfg2 or cfg3" 2>&1 | tail -2
QSIM_QFT_LOAD=cpa timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -k "qft or hadamard or cfg2 or cfg3" 2>&1 | tail -2
for L in auto tma cpa; do
for A in 10 9 7; do
  if [ $L = auto ]; then unset QSIM_QFT_LOAD; else export QSIM_QFT_LOAD=$L; fi
  QSIM_QFT_AMAX=$A timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_a$A.log 2>&1
  python - <<PY
import json; d=json.loads(open("gpurun_out/bench_a$A.log").read().strip().splitlines()[-1])
print("$L amax=$A", "ms=%.3f"%d["ms_per_step"], list(d["kernels"].keys()), "passes", d["step_launches_ms"])
PY
done
done
