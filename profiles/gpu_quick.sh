timeout 900 python -m pytest tests/test_device_fast.py tests/test_ts_mma.py tests/test_device_check.py -x -q > gpurun_out/quick_tests.log 2>&1
timeout 300 python bench.py --steps 20 --no-cpu --secondary "dag_mdb_b8192,hypergrid_tb_b16,hypergrid_subtb_b65536" > gpurun_out/bench2.log 2>&1
python profiles/rollout_phases.py > gpurun_out/phases_hg2.json 2>&1; cat gpurun_out/phases_hg2.json
python -c "
import json; d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value']); print({k:round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items()}); print({k:(v.get('ms_per_iter'), v.get('kernels_ms_per_iter')) for k,v in d['secondary'].items()})"
tail -3 gpurun_out/quick_tests.log
