for v in ab/*.so; do echo "$v"; cp $v paper_2511_16592_b200/libgfnx.so; timeout 300 python bench.py --steps 20 --no-cpu --no-e2e --secondary "dag_mdb_b8192" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print(d['secondary']['dag_mdb_b8192']['ms_per_iter'], d['secondary']['dag_mdb_b8192']['kernels_ms_per_iter'])"; done
