# A/B of library builds under ab/ on the headline bench, kernel breakdown (diagnostic)
for v in ab/*.so; do echo "$v"; cp $v paper_2511_16592_b200/libgfnx.so; timeout 300 python bench.py --steps 20 --no-cpu --no-e2e --secondary "" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print(round(d['value']/1e6,3), round(d['ms_per_step'],4), {k:round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items()})"; done
