# A/B of the gate-list pass: parity with the new build, configs timings new vs .ab/libqsim_old.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
L=paper_quant_ph_0201042_b200/libqsim.so
for round in 1 2; do
timeout 600 python tools/bench_configs.py ${CFGS:-4 3n 0} > gpurun_out/cfg_new$round.jsonl 2> gpurun_out/cfg_new.err; echo "cfg new rc=$?"
cp $L .ab/libqsim_new.so; cp .ab/libqsim_old.so $L
timeout 600 python tools/bench_configs.py ${CFGS:-4 3n 0} > gpurun_out/cfg_old$round.jsonl 2> gpurun_out/cfg_old.err; echo "cfg old rc=$?"
cp .ab/libqsim_new.so $L
done
