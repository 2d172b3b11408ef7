# Per-instruction stall sampling of one late-iteration launch of the fused hypergrid rollout
# (diagnostic): ncu source page (SASS + CUDA line) of k_fast_rollout_ts in the bench command
K=${1:-40}
ncu --set full --clock-control none --import-source on -k regex:"k_fast_rollout_ts" --launch-skip 30 -c 1 \
  -o /tmp/rsrc -f python bench.py --steps $K --warmup 5 --no-cpu --no-e2e --no-steady --no-sweep --secondary "" > gpurun_out/rsrc.log 2>&1
ncu -i /tmp/rsrc.ncu-rep --page source --csv --print-source sass > gpurun_out/rsrc_sass.csv 2>&1
ncu -i /tmp/rsrc.ncu-rep --page source --csv --print-source cuda > gpurun_out/rsrc_cuda.csv 2>&1
ncu -i /tmp/rsrc.ncu-rep --page details --csv > gpurun_out/rsrc_details.csv 2>&1
ls -la gpurun_out/rsrc*
