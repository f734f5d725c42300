# ncu --set full of the other hot kernels: gate-list passes (configs[4] n = 30 heavy pass,
# configs[3] sigma = 1e-3 H pass), the generalised QFT pass and the MODEXP ring
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cap() {  # name kernel-regex skip cmd...
  local name=$1 k=$2 s=$3; shift 3
  timeout 300 "$@" > gpurun_out/plain_$name.log 2>&1 || { echo "$name plain failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 1 -o gpurun_out/prof_$name "$@" > gpurun_out/ncu_$name.log 2>&1
  echo "$name ncu rc=$?"
  ncu -i gpurun_out/prof_$name.ncu-rep --page details > gpurun_out/prof_${name}_details.txt 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/prof_${name}_raw.csv 2>&1
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_${name}_src.csv 2>&1
  rm -f gpurun_out/prof_$name.ncu-rep
}
cap ops_pass k_ops_pass 0 python tools/run_cfg.py 4m
cap ops_pp k_ops_pp 0 python tools/run_cfg.py 4m
cap qft_gen k_qft_gen 0 python tools/run_cfg.py 3n
cap perm_ring k_perm_ring 0 python tools/run_cfg.py 3
cap grover_regs k_grover_regs 0 python tools/run_cfg.py 1
cap probs_warp k_probs_warp 0 python tools/run_cfg.py 3
