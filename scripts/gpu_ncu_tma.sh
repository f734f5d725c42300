cd $GRAFT_REPO_ROOT
CMD="python bench.py --profile-only --steps 1 --warmup 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile -c 3 \
    -o gpurun_out/prof_tma $CMD > gpurun_out/ncu_tma.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_tma.log
