# ncu capture of the fused tile kernel (QFT pass) at n=28 + launch list of the bench step
cd $GRAFT_REPO_ROOT
CMD="python bench.py --profile-only --steps 1 --warmup 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_pass -c 3 \
    -o gpurun_out/prof_tile $CMD > gpurun_out/ncu_tile.log 2>&1
echo "ncu rc=$?"
tail -5 gpurun_out/ncu_tile.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile-only --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
