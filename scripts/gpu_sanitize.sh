# one compute-sanitizer tool per gpurun call: TOOL=racecheck|synccheck|memcheck
cd $GRAFT_REPO_ROOT
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/san_$TOOL.log 2>&1
echo "rc=$?"; tail -25 gpurun_out/san_$TOOL.log
