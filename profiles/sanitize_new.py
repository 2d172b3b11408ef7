"""compute-sanitizer driver for the round-2 kernels (walks, teacher-forced batches, MC,
pearson, EB-GFN, deterministic rollout, lockstep DB / ragged / AR): small sizes.
usage: compute-sanitizer --tool memcheck python profiles/sanitize_new.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402


def walks(e, t):
    tr = engine.Trainer(e, t)
    tr.forward_rollout(0, 1.0)
    terms = tr.batch(("terminal_state",))["terminal_state"].copy()
    tr.backward_rollout(terms, (1, 2))
    tr.compute_grads()
    keys = np.arange(2 * 8, dtype=np.uint64).reshape(8, 2)
    tr.mc_terminal_logprob(terms[:8], keys, 3)
    tr.close()


for check in (False, True):
    for e, t in [(abi.env_desc(abi.HYPERGRID, hg_dim=2, hg_side=6), abi.train_desc(abi.HYPERGRID, batch=128)),
                 (abi.env_desc(abi.DAG, dag_d=4), abi.train_desc(abi.DAG, batch=128)),
                 (abi.env_desc(abi.ISING, is_side=3), abi.train_desc(abi.ISING, batch=130, hidden=(256, 256))),
                 (abi.env_desc(abi.BITSEQ, bs_n_bits=16, bs_k=8, bs_scheme=1),
                  abi.train_desc(abi.BITSEQ, batch=128, objective="db"))]:
        if check:
            t.precision = abi.PREC_FP64_CHECK
        walks(e, t)
        print("walks ok", e.kind, check, flush=True)

e, t = abi.config("hypergrid_db_b65536", batch=2048)
t.deterministic = 1
tr = engine.Trainer(e, t)
tr.run(0, 3)
tr.close()
print("deterministic ok", flush=True)

e = abi.env_desc(abi.ISING, is_side=2, is_sigma=0.3)
t = abi.train_desc(abi.ISING, batch=8, hidden=(16,), iterations=5)
t.precision = abi.PREC_FP64_CHECK
t.learned_backward = 1
tr = engine.Trainer(e, t)
tr.eb_init(engine.eb_desc(data_samples=50, gibbs_burn_in=20, k=3, data_batch=8))
tr.eb_run(0, 3)
tr.close()
print("eb ok", flush=True)

e = abi.env_desc(abi.BITSEQ, bs_n_bits=16, bs_k=8)
t = abi.train_desc(abi.BITSEQ, batch=128)
tr = engine.Trainer(e, t)
tr.pearson(0, 2)
tr.close()
print("pearson ok", flush=True)
