# A/B of a whole older tree (ab/<name>/, its own bench.py + libgfnx.so) against the current
# one on the headline bench (50 steps), kernel breakdown (diagnostic)
run() {
  (cd $1 && timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-e2e --no-steady --no-sweep --secondary "" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.load(sys.stdin); print('$1', round(d['value']/1e6,3), round(d['ms_per_step'],4), {k:round(v['ms_total']/v['launches'],4) for k,v in d['kernels'].items()})")
}
for i in 1 2; do for t in "$@"; do run $t; done; done
