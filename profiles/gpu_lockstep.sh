timeout 600 python -m pytest tests/test_device_fast.py -x -q -k "lockstep" > gpurun_out/ls_tests.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --secondary "bitseq_tb_b16384,ising_tb_b32768" > gpurun_out/bench_ls.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_ls.log').read().strip().splitlines()[-1])
for k,v in d['secondary'].items(): print(k, v.get('trajectories_per_s'), v.get('ms_per_iter'), v.get('kernels_ms_per_iter'))"
tail -2 gpurun_out/ls_tests.log
