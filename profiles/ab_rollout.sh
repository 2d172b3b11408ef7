# A/B of library builds under ab/ on the hypergrid rollout (diagnostic)
for v in ab/*.so; do echo "$v"; cp $v paper_2511_16592_b200/libgfnx.so; python profiles/rollout_phases.py ${1:-hypergrid_db_b65536} 2>&1 | python -c "
import json,sys; d=json.load(sys.stdin); print({k:d[k] for k in ('loop_barrier','layer1','hidden_mma','hidden_epilogue','head_mma','sample_step','rollout_ms_per_iter')})"; done
