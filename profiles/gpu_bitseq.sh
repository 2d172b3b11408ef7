ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bitseq.csv python profiles/run_config.py bitseq_tb_b16384 --iters 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_ls_sample|k_ls_wgrad" --launch-skip 130 --launch-count 12 -o gpurun_out/bitseq_full python profiles/run_config.py bitseq_tb_b16384 --iters 3 > gpurun_out/ncu_bitseq.log 2>&1
tail -2 gpurun_out/ncu_bitseq.log
