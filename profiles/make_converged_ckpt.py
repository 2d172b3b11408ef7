"""Train hypergrid 20^4 DB at B = 65536 on the device until the policy's exact terminal
marginal is close to R/Z, then save a GFNCKPT1 checkpoint for bench.py's steady-state leg
(mean trajectory length under the target policy is 39.0)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16592_b200 import abi, engine  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "hypergrid_db_converged.ckpt")
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
e, t = abi.config("hypergrid_db_b65536")
t.iterations = 1_000_000
tr = engine.Trainer(e, t)
log = []
t0 = time.time()
done = 0
while done < iters:
    n = min(250, iters - done)
    tr.run(done, n)
    done += n
    _, tv = tr.exact_terminal_marginal(20 ** 4)
    L = float(tr.batch(["lengths"])["lengths"].mean())
    log.append({"iter": done, "tv_exact": tv, "mean_traj_len": L, "wall_s": round(time.time() - t0, 1)})
    print(json.dumps(log[-1]), flush=True)
tr.save_checkpoint(out, done)
print(json.dumps({"saved": out, "iters": done, "final": log[-1]}))
