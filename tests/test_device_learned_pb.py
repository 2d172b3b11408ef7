"""GPU: the learned backward policy (LossConfig::learned_backward, objectives.cpp:57-70 / 186-226)
in fp64 check mode.

log P_B(s_t | s_{t+1}) comes from the policy's backward head at s_{t+1} (mlp_forward_tape's bwd
leaves, nn.cpp:111-121) under the backward action mask: k_check_fwd's bwd pass over the
s_{t+1} rows, the objectives' -g into those rows, k_check_bwd through the bwd head + trunk and
a second row set in k_check_wgrad. Compared with the compiled reference (its own
mlp_forward_tape + build_loss + Tape::backward) on the same batch: loss and every gradient
element to 1e-9 (the two row sets sum the trunk gradient in a different association order
than the reference's shared rows; ulp-level), Adam-updated parameters as well.
The bf16 paths keep the uniform P_B and reject learned_backward with config_error.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu

CASES = [
    ("hypergrid_tb", lambda: (abi.env_desc(abi.HYPERGRID, hg_dim=3, hg_side=5),
                              abi.train_desc(abi.HYPERGRID, batch=16, objective="tb", seed=2))),
    ("hypergrid_db", lambda: (abi.env_desc(abi.HYPERGRID, hg_dim=2, hg_side=6),
                              abi.train_desc(abi.HYPERGRID, batch=16, objective="db", seed=3))),
    ("hypergrid_subtb", lambda: (abi.env_desc(abi.HYPERGRID, hg_dim=2, hg_side=6),
                                 abi.train_desc(abi.HYPERGRID, batch=12, objective="subtb", seed=4))),
    ("dag_mdb", lambda: (abi.env_desc(abi.DAG, dag_d=4, dag_score=abi.BGE),
                         abi.train_desc(abi.DAG, batch=16, objective="mdb", seed=5))),
    ("bitseq_tb", lambda: (abi.env_desc(abi.BITSEQ, bs_n_bits=16, bs_k=4),
                           abi.train_desc(abi.BITSEQ, batch=16, objective="tb", seed=6))),
    ("ising_db", lambda: (abi.env_desc(abi.ISING, is_side=3),
                          abi.train_desc(abi.ISING, batch=8, objective="db", seed=7, hidden=(64, 64)))),
]


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name,mk", CASES)
def test_learned_backward_matches_reference(name, mk):
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = mk()
    t.learned_backward = 1
    t.precision = abi.PREC_FP64_CHECK
    d = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    ref.set_params(*d.params())
    for it in (0, 1, 2):
        eps = 0.3
        d.forward_rollout(it, eps)
        ref.rollout(it, eps)
        bd, br = d.batch(), ref.batch(d.T)
        for k in ("lengths", "fwd_actions", "log_rewards"):
            assert np.array_equal(bd[k], br[k]), (name, it, k)
        ld, lr = d.compute_grads(), ref.compute_grads()
        (gd, zd), (gr, zr) = d.grads(), ref.grads()
        assert abs(ld - lr) <= 1e-10 * max(1.0, abs(lr)), (name, it, ld, lr)
        assert _rel(gd, gr) <= 1e-9, (name, it, _rel(gd, gr))
        assert abs(zd - zr) <= 1e-10 * max(1.0, abs(zr))
        bw = slice(*_bwd_head(d, t))  # the backward head really receives gradient
        assert np.abs(gr[bw]).max() > 0 and _rel(gd[bw], gr[bw]) <= 1e-9
        ref.apply_adam(1e-3)
        d.set_params(*ref.params())
    d.close()


def _bwd_head(d, t):
    """[start, end) of the bwd head (W then b) in MlpParams::tensors() order (nn.cpp:8-19)."""
    shape = d.shape
    H = t.hidden[t.num_hidden - 1]
    n = d.n_params
    nflow = H + 1
    end = n - nflow
    start = end - (H * shape.num_backward_actions + shape.num_backward_actions)
    return start, end


def test_learned_backward_rejected_on_bf16_paths():
    e = abi.env_desc(abi.HYPERGRID, hg_dim=3, hg_side=5)
    t = abi.train_desc(abi.HYPERGRID, batch=16, objective="tb")
    t.learned_backward = 1
    with pytest.raises(engine.config_error, match="learned backward"):
        engine.Trainer(e, t)


@pytest.mark.parametrize("name,mk", [CASES[0], CASES[3], CASES[4], CASES[5]])
def test_learned_backward_walks_and_mc_match_reference(name, mk):
    """backward_rollout sampling from the learned backward head (env_core.hpp:331-359) and
    mc_terminal_logprob scored with it (exact.hpp:229-241, score_trajectories learned branch),
    against the reference on the same parameters and keys."""
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = mk()
    t.learned_backward = 1
    t.precision = abi.PREC_FP64_CHECK
    d = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    d.run(0, 5)  # a non-uniform backward head
    ref.set_params(*d.params())
    d.forward_rollout(7, 1.0)
    terms = d.batch(("terminal_state",))["terminal_state"].copy()
    key = (0xABCDEF, 0x12345)
    d.backward_rollout(terms, key)
    ref.backward_rollout(terms, key)
    bd, br = d.batch(), ref.batch(d.T)
    for k in ("lengths", "fwd_actions", "log_rewards", "log_pb"):
        assert np.array_equal(bd[k], br[k]), (name, k)
    rng = np.random.default_rng(1)
    keys = rng.integers(0, 2**63, size=(len(terms), 2), dtype=np.uint64)
    dev = d.mc_terminal_logprob(terms, keys, 4)
    want = np.array([ref.mc_logprob(terms[i], keys[i], 4) for i in range(len(terms))])
    assert np.max(np.abs(dev - want)) <= 1e-9 * max(1.0, np.max(np.abs(want))), np.max(np.abs(dev - want))
    d.close()
