# A/B of whole trees (ab/<name>/ with its own bench.py + libgfnx.so, and .) on secondary configs
# usage: bash profiles/ab_tree_cfg.sh bitseq_tb_b16384,ising_tb_b32768 ab/r2 .
cfg=$1; shift
for i in 1 2; do for t in "$@"; do (cd $t && timeout 600 python -c "
import sys; sys.path.insert(0, '.')
import bench
r = bench.secondary_runs('$cfg'.split(','), 10, 2, 0)
for k, v in r.items(): print('$t', k, v.get('error') or (round(v['ms_per_iter'], 4), {a: b for a, b in v['kernels_ms_per_iter'].items() if b > 0.04}))
"); done; done
