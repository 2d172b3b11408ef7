# ncu --set full of the hot kernels of BASELINE configs #3, #4, #5 (iteration 2 of
# profiles/run_config.py --iters 3), summarised into profiles/<round>_ncu_<config>.md
# usage: bash profiles/gpu_profile_configs.sh r2
R=${1:-r2}
run() {  # config, kernel regex, launches per iteration matching the regex
  ncu --set full --clock-control none --import-source on -k regex:"$2" --launch-skip $((2 * $3)) --launch-count $3 \
    -o gpurun_out/full_${1}_$R python profiles/run_config.py $1 --iters 3 > gpurun_out/ncu_${1}_$R.log 2>&1
  NCU_NO_TRAFFIC=1 python profiles/summarize_ncu.py gpurun_out/full_${1}_$R.ncu-rep gpurun_out/${R}_ncu_${1}.md > /dev/null
  bash profiles/ncu_brief.sh gpurun_out/full_${1}_$R.ncu-rep > gpurun_out/${R}_ncu_${1}_brief.txt 2>&1
  tail -1 gpurun_out/ncu_${1}_$R.log
}
run bitseq_tb_b16384 "k_gemm|k_ls_(sample|wgrad|layer1)" 64
run ising_tb_b32768 "k_ls_persist|k_gemm|k_ls_wgrad" 7
run dag_mdb_b8192 "k_fast_(rollout|bwd|wgrad|loss)|k_row_stats" 5
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/  # keep the merge-back under 64 MiB
