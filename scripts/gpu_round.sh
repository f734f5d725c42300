#!/bin/bash
# Full GPU check: parity suite, bench line, Shor Table 5 reproduction.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | cut -c1-1500
timeout 600 python tools/bench_configs.py 2 3 > gpurun_out/configs.jsonl 2>&1; echo "configs rc=$?"
if [ "${SHOR:-1}" = 1 ]; then
  timeout 1200 python tools/shor_table5.py 100 2002 > gpurun_out/shor_table5.jsonl 2> gpurun_out/shor_table5.err
  echo "table5 rc=$?"
fi
