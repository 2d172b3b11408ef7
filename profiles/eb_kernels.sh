# per-kernel device time of 3 EB-GFN iterations (Ising 10x10, B = 256, 4x256; ncu launch list, diagnostic)
ncu --metrics gpu__time_duration.sum --csv --clock-control none -c 300 python -c "
import sys; sys.path.insert(0, '.')
from paper_2511_16592_b200 import abi, engine
e = abi.env_desc(abi.ISING, is_side=10, is_sigma=0.2)
t = abi.train_desc(abi.ISING, batch=256, iterations=1000000)
tr = engine.Trainer(e, t)
tr.eb_init(engine.eb_desc(data_batch=256))
tr.eb_run(0, 3)
tr.synchronize()
" 2>/dev/null | grep -v "^==" | python3 -c "
import csv, sys, collections
r = list(csv.reader(sys.stdin))
h = r[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(float); cnt = collections.Counter()
for row in r[1:]:
    try: v = float(row[vi].replace(',', ''))
    except (ValueError, IndexError): continue
    n = row[ki].split('(')[0][-60:]
    agg[n] += v; cnt[n] += 1
for n, v in sorted(agg.items(), key=lambda x: -x[1])[:12]: print(round(v / 3e3, 1), 'us/iter', cnt[n] // 3, n)
"
