# Per-instruction stall sampling of one k_ls_persist launch (Ising config #4; diagnostic)
ncu --set full --clock-control none --import-source on -k regex:"k_ls_persist" --launch-skip 2 --launch-count 1 \
  -o /tmp/psrc -f python profiles/run_config.py ising_tb_b32768 --iters 3 > gpurun_out/psrc.log 2>&1
ncu -i /tmp/psrc.ncu-rep --page source --csv --print-source sass > gpurun_out/psrc_sass.csv 2>&1
ncu -i /tmp/psrc.ncu-rep --page details --csv > gpurun_out/psrc_details.csv 2>&1
python profiles/persist_phases.py > gpurun_out/psrc_phases.log 2>&1
