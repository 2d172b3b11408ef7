# full bench line + ncu launch list + one ncu --set full capture of the hot kernels (round profile)
R=${1:-r1}
timeout 900 python bench.py > gpurun_out/bench_full_$R.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --secondary "" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fast_(rollout|bwd|wgrad|loss)|k_row_stats" --launch-skip 40 --launch-count 5 -o gpurun_out/full_$R python profiles/run_config.py hypergrid_db_b65536 --iters 12 > gpurun_out/ncu_full_$R.log 2>&1
tail -2 gpurun_out/ncu_full_$R.log
