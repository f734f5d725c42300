#!/bin/bash
# Row f3 on the GPU: Shor parity tests, then the Table 5 reproduction.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shor.py -x -q > gpurun_out/shor_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/shor_tests.log
timeout 1200 python tools/shor_table5.py 100 2002 > gpurun_out/shor_table5.jsonl 2> gpurun_out/shor_table5.err
echo "table5 exit $?"
tail -3 gpurun_out/shor_tests.log
