ncu --set full --clock-control none --import-source on -k regex:"k_gemm" --launch-skip 63 --launch-count 2 -o gpurun_out/bitseq_dlog python profiles/run_config.py bitseq_tb_b16384 --iters 2 > gpurun_out/ncu_bitseq2.log 2>&1
tail -2 gpurun_out/ncu_bitseq2.log
