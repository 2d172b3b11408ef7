# Round profile: full bench line, reference arm, ncu launch list of the bench's own command,
# and one ncu --set full capture of the hot kernels of timed iteration W+J of the SAME command
# (so roofline.traffic is a launch of the timed region). usage: bash profiles/gpu_profile.sh r2
R=${1:-r2}; W=5; K=50; J=25
timeout 900 python bench.py --steps $K --warmup $W > gpurun_out/bench_full_$R.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv \
  python bench.py --steps $K --warmup $W --no-cpu --no-e2e --no-steady --no-sweep --secondary "" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fast_(rollout|bwd|wgrad)" \
  --launch-skip $((3 * (W + J))) --launch-count 3 -o gpurun_out/full_$R \
  python bench.py --steps $K --warmup $W --no-cpu --no-e2e --no-steady --no-sweep --secondary "" > gpurun_out/ncu_full_$R.log 2>&1
ROWS=$(python -c "import json; d=json.loads(open('gpurun_out/bench_full_$R.log').read().strip().splitlines()[-1]); print(d['roofline']['algorithmic_per_launch']['rows'])")
python profiles/summarize_ncu.py gpurun_out/full_$R.ncu-rep gpurun_out/${R}_ncu_summary.md $ROWS \
  "ncu --set full, bench.py --steps $K --warmup $W timed iteration W+$J (rows = mean rows per timed iteration)"
tail -2 gpurun_out/ncu_full_$R.log
# (summarize_ncu.py writes gpurun_out/ncu_traffic.json next to the summary: copy it into profiles/)
bash profiles/ncu_brief.sh gpurun_out/full_$R.ncu-rep > gpurun_out/${R}_ncu_brief.txt 2>&1
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/  # keep the merge-back under 64 MiB
