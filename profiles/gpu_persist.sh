ncu --set full --clock-control none --import-source on -k regex:"k_ls_persist" --launch-skip 2 --launch-count 1 -o gpurun_out/persist python profiles/run_config.py ising_tb_b32768 --iters 3 > gpurun_out/ncu_persist.log 2>&1
tail -1 gpurun_out/ncu_persist.log
