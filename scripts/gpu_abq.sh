# A/B of k_qft13 builds: per-pass times of the in-tree build vs .ab/libqsim_head.so, alternating
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for lib in "" .ab/libqsim_head.so; do
    for n in ${NS:-28 29}; do
      echo "lib=${lib:-new} $(QSIM_LIB=$lib timeout 300 python tools/probe_qft3.py $n qft 2>&1 | tail -1 | cut -c1-250)"
    done
  done
done
