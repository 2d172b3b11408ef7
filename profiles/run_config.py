#!/usr/bin/env python
"""Run a few training iterations of one BASELINE config (ncu / sanitizer driver).

  python profiles/run_config.py bitseq_tb_b16384 --iters 3 [--batch 16384]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_16592_b200 import abi, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--batch", type=int, default=None)
args = ap.parse_args()
kw = {} if args.batch is None else {"batch": args.batch}
e, t = abi.config(args.config, **kw)
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, args.iters)
tr.synchronize()
print("loss", tr.iteration_loss if hasattr(tr, "iteration_loss") else "ok")
tr.close()
