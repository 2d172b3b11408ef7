# A/B of library builds under ab/ on secondary configs (device-timed, kernel breakdown; diagnostic)
# usage: bash profiles/ab_config.sh bitseq_tb_b16384[,ising_tb_b32768]
for v in ab/*.so; do echo "$v"; cp $v paper_2511_16592_b200/libgfnx.so; timeout 300 python -c "
import json, sys; sys.path.insert(0, '.')
import bench
r = bench.secondary_runs('$1'.split(','), 10, 2, 0)
for k, v in r.items(): print(k, v.get('error') or (round(v['ms_per_iter'], 4), {a: b for a, b in v['kernels_ms_per_iter'].items() if b > 0.05}))
"; done
