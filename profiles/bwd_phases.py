#!/usr/bin/env python
"""Per-tile phase clocks of k_fast_bwd (thread 0 of each CTA; diagnostic).

  python profiles/bwd_phases.py [config]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402

e, t = abi.config(sys.argv[1] if len(sys.argv) > 1 else "hypergrid_db_b65536")
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, 30)
tr.synchronize()
tr.phase_timers(1)
tr.profile(True)
tr.run(30, 10)
tr.synchronize()
ph = tr.phase_timers(2)
prof = tr.profile_read()
tiles = max(ph["bwd_tiles"], 1)
out = {k: round(ph[k] / tiles / 1965.0, 3) for k in ("bwd_rowload", "bwd_wait_dlogits", "bwd_head", "bwd_dz2", "bwd_w2mma_db2", "bwd_dz1")}
out["tiles_per_cta_per_iter"] = tiles / 10 / 148
out["bwd_ms_per_iter"] = prof.get("k_fast_bwd", (0, 1))[0] / 10
out["wgrad_ms_per_iter"] = prof.get("k_fast_wgrad", (0, 1))[0] / 10
print(json.dumps(out, indent=1))
tr.close()
