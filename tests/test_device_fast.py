"""GPU: the bf16 tcgen05 fast path of libgfnx against the oracle.

* eps = 1 makes every legal action exactly 1/#legal in the reference sampler, so the
  fast rollout must reproduce the oracle's trajectories BIT-EXACTLY regardless of the
  bf16 policy (actions, lengths, terminal states, log-rewards, log P_B, MDB deltas).
* Loss / gradient / per-row log pi parity on the same batch, with the stated tolerances, is in
  tests/test_device_parity.py (bf16 operand model and fp64, benchmark batch sizes).
* A full iteration (Adam) moves the parameters like the oracle's step.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu

CASES = [
    ("hypergrid_tb_b16", dict()),
    ("hypergrid_db_b65536", dict(batch=1024)),
    ("hypergrid_subtb_b65536", dict(batch=512)),
    ("dag_mdb_b8192", dict(batch=256)),
]


def _pair(name, **kw):
    e, t = abi.config(name, **kw)
    return e, t


def _same_batch(bd, bo):
    for k in ("lengths", "fwd_actions", "bwd_actions", "log_rewards", "log_pb", "delta",
              "terminal_state"):
        assert np.array_equal(bd[k], bo[k]), k


@pytest.mark.parametrize("name,kw", CASES)
def test_fast_rollout_bitexact_at_eps1(name, kw):
    e, t = _pair(name, **kw)
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    for it in (0, 3):
        d.forward_rollout(it, 1.0)
        o.rollout(it, 1.0)
        _same_batch(d.batch(), o.batch())
    d.close()


def _grad_close(gd, go):
    err = np.linalg.norm(gd - go) / max(np.linalg.norm(go), 1e-30)
    cos = float(gd @ go / max(np.linalg.norm(gd) * np.linalg.norm(go), 1e-30))
    return err, cos


@pytest.mark.parametrize("name,kw", CASES)
def test_fused_rollout_forward_matches_recomputed_forward(name, kw):
    """The rollout emits every sampled row's activations (fused training forward). After
    set_params the same batch is re-scored by the separate training-forward kernel; both
    must give the same loss and gradient up to fp32 summation order in layer 1."""
    e, t = _pair(name, **kw)
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    p, z = o.params()
    d.set_params(p, z)
    d.forward_rollout(1, o.schedule("explore", 1))
    l_fused = d.compute_grads()
    g_fused, dz_fused = d.grads()
    d.set_params(p, z)  # same weights: invalidates the rollout's activations
    l_re = d.compute_grads()
    g_re, dz_re = d.grads()
    assert abs(l_fused - l_re) <= 1e-3 * abs(l_re) + 1e-6, (l_fused, l_re)
    err, cos = _grad_close(g_fused, g_re)
    assert err < 3e-2 and cos > 0.9995, (err, cos)
    d.close()


def test_fast_iteration_tracks_oracle_step():
    e, t = _pair("hypergrid_tb_b16")
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    p0, z0 = o.params()
    d.set_params(p0, z0)
    d.forward_rollout(0, 0.0)
    o.replay(d.batch()["fwd_actions"])
    d.train_step(1e-3)
    o.compute_grads()
    o.apply_adam(1e-3)
    pd, zd = d.params()
    po, zo = o.params()
    go, _ = o.grads()
    # the first Adam step is ~lr * sign(g): compare where the gradient is not ~0 (elsewhere
    # bf16 vs fp64 rounding may flip the sign of a vanishing component)
    m = np.abs(go) > 1e-2 * np.abs(go).max()
    step_d, step_o = (pd - p0)[m], (po - p0)[m]
    err, cos = _grad_close(step_d, step_o)
    assert err < 5e-2 and cos > 0.998, (err, cos)
    assert abs(zd - zo) < 1e-4
    d.close()


def test_fast_run_loop_and_launch_count():
    e, t = _pair("hypergrid_db_b65536", batch=4096)
    d = engine.Trainer(e, t)
    n0 = d.kernel_launches()
    losses = d.run(0, 5, read_losses=True)
    assert np.all(np.isfinite(losses))
    assert d.kernel_launches() - n0 >= 5 * 8
    d.close()


def test_iteration_async_slots_match_batch_export():
    e, t = _pair("hypergrid_db_b65536", batch=2048)
    d = engine.Trainer(e, t)
    d.iteration_async(0, 0)
    d.iteration_async(1, 1)
    it0, loss0, r0 = d.slot_wait(0)
    it1, loss1, r1 = d.slot_wait(1)
    assert (it0, it1) == (0, 1) and np.isfinite(loss0) and np.isfinite(loss1)
    b = d.batch()  # resident batch = iteration 1
    for k in ("lengths", "log_rewards", "terminal_state"):
        assert np.array_equal(r1[k], b[k]), k
    d.close()


# ---- fixed-length (lockstep) fast path: bit-sequence NAR k = 8 (config #3 shape) and
# Ising (config #4 shape, 4 x 256 MLP)
def _bitseq(n_bits, batch):
    e = abi.env_desc(abi.BITSEQ, bs_n_bits=n_bits, bs_k=8)
    t = abi.train_desc(abi.BITSEQ, batch=batch, objective="tb")
    return e, t


def _ising(side, batch):
    e = abi.env_desc(abi.ISING, is_side=side, is_sigma=0.2)
    t = abi.train_desc(abi.ISING, batch=batch, objective="tb")
    return e, t


LOCKSTEP_EPS1 = [("bitseq", lambda: _bitseq(120, 128)), ("ising", lambda: _ising(10, 128))]


@pytest.mark.parametrize("name,mk", LOCKSTEP_EPS1)
def test_lockstep_fast_rollout_bitexact_at_eps1(name, mk):
    e, t = mk()
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    for it in (0, 2):
        d.forward_rollout(it, 1.0)
        o.rollout(it, 1.0)
        _same_batch(d.batch(), o.batch())
    d.close()


@pytest.mark.parametrize("name,mk", [("bitseq", lambda: _bitseq(120, 16384)), ("ising", lambda: _ising(10, 16384))])
def test_lockstep_sampler_matches_policy_distribution(name, mk):
    """eps = 0: first actions of a large batch (all from s0) follow softmax(policy(s0))."""
    e, t = mk()
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    p, z = o.params()
    p = 4.0 * p  # sharpen the policy so the test has power
    o.set_params(p, z)
    d.set_params(p, z)
    d.forward_rollout(0, 0.0)
    a0 = d.batch()["fwd_actions"][:, 0]
    obs, mask = o.obs_after(np.zeros(0, dtype=np.int32))
    lg, _ = o.mlp_forward(obs[None])
    lg = np.where(mask > 0, lg[0], -np.inf)
    pr = np.exp(lg - lg.max())
    pr /= pr.sum()
    cnt = np.bincount(a0, minlength=len(pr)).astype(np.float64)
    if name == "bitseq":  # marginals over slot and word (A = 15 x 256)
        bins = [(cnt.reshape(-1, 256).sum(1), pr.reshape(-1, 256).sum(1)),
                (cnt.reshape(-1, 256).sum(0), pr.reshape(-1, 256).sum(0))]
    else:
        bins = [(cnt, pr)]
    n = len(a0)
    for c, q in bins:
        keep = n * q >= 5
        chi2 = float((((c - n * q) ** 2) / np.maximum(n * q, 1e-30))[keep].sum())
        dof = int(keep.sum()) - 1
        assert chi2 < dof + 6 * np.sqrt(2 * dof), (chi2, dof)
        assert c[~keep].sum() <= max(20, 3 * n * q[~keep].sum())
    d.close()


@pytest.mark.parametrize("name,mk,T", [("bitseq", lambda: _bitseq(120, 1024), 15),
                                      ("ising", lambda: _ising(10, 1024), 100)])
def test_lockstep_fast_iterations_run(name, mk, T):
    e, t = mk()
    d = engine.Trainer(e, t)
    losses = d.run(0, 3, read_losses=True)
    assert np.all(np.isfinite(losses))
    b = d.batch()
    assert np.all(b["lengths"] == T)
    d.close()


def test_fused_rows_account_for_every_step():
    """Row counters published by the rollout (no scan) equal sum(L) of the exported batch,
    across iterations (the counters are reset per rollout)."""
    e, t = _pair("hypergrid_db_b65536", batch=3000)
    d = engine.Trainer(e, t)
    for it in range(3):
        r0 = d.counters()[0]
        d.iteration(it)
        d.synchronize()
        r1 = d.counters()[0]
        assert r1 - r0 == int(d.batch()["lengths"].sum())
    d.close()
