#!/usr/bin/env python
"""Per-phase clock breakdown of the persistent rollout kernel (diagnostic).

  python profiles/rollout_phases.py [config] [--batch B] [--warmup W] [--iters N]
Prints, per tile-step of one CTA, the microseconds spent in each phase (clock64 at the
SM clock, summed over CTAs then divided by the tile-steps), plus slot occupancy.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="hypergrid_db_b65536")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--warmup", type=int, default=30)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--mhz", type=float, default=1965.0)
args = ap.parse_args()
kw = {} if args.batch is None else {"batch": args.batch}
e, t = abi.config(args.config, **kw)
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, args.warmup)
tr.synchronize()
tr.phase_timers(1)
tr.profile(True)
tr.run(args.warmup, args.iters)
tr.synchronize()
ph = tr.phase_timers(2)
prof = tr.profile_read()
steps = ph["tile_steps"]
out = {k: round(v / steps / args.mhz, 3) for k, v in ph.items() if k not in ("tile_steps", "active_slot_steps")}
out["tile_steps_per_cta_per_iter"] = steps / args.iters / 148
out["slot_occupancy"] = ph["active_slot_steps"] / (128 * steps)
out["rollout_ms_per_iter"] = prof.get("k_fast_rollout", (0, 1))[0] / args.iters
print(json.dumps(out, indent=1))
tr.close()
