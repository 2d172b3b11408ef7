"""GPU: backward walks and teacher-forced batches on the device.

* gfnx_backward_rollout = backward_rollout under the uniform backward policy
  (env_core.hpp:314-370) followed by rollout_from_actions (:166-229): the device walk draws
  from the reference's Threefry stream, so the batch (forward actions, lengths, log P_B,
  log-rewards, terminals) is compared BIT-EXACTLY with the compiled reference's
  backward_rollout on the same terminals and key, every env, both precisions; the training
  pass on that batch then agrees to 1e-9 (fp64 check mode) / rtol 1e-4 (bf16, the loss
  tolerance of DESIGN.md §2).
* gfnx_rollout_from_actions replays the reference's own forward batch.
* gfnx_mc_terminal_logprob for every env: fp64 check mode against the reference's
  mc_terminal_logprob (exact.hpp:229-241) to 1e-9, bf16 to the bf16 policy tolerance.
Bitseq at k = 8 (the bf16 lockstep path) cannot run in the reference (vocab cap 64,
sequences.cpp:192-193): there the bf16 batch is compared with the device's fp64 check mode,
which is pinned against the reference at k = 6.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu

FIELDS = ("lengths", "fwd_actions", "log_rewards", "log_pb", "terminal_state")
REF_FIELDS = ("lengths", "fwd_actions", "log_rewards", "log_pb")


def _cfg(name, check):
    if name == "hypergrid":
        e = abi.env_desc(abi.HYPERGRID, hg_dim=3, hg_side=6)
        t = abi.train_desc(abi.HYPERGRID, batch=128, objective="tb", seed=3)
    elif name == "hypergrid_db":
        e = abi.env_desc(abi.HYPERGRID, hg_dim=4, hg_side=8)
        t = abi.train_desc(abi.HYPERGRID, batch=256, objective="db", seed=4)
    elif name == "dag_mdb":
        e = abi.env_desc(abi.DAG, dag_d=4, dag_score=abi.BGE)
        t = abi.train_desc(abi.DAG, batch=128, objective="mdb", seed=5)
    elif name == "bitseq_k6":
        e = abi.env_desc(abi.BITSEQ, bs_n_bits=24, bs_k=6)
        t = abi.train_desc(abi.BITSEQ, batch=128, objective="tb", seed=6)
    elif name == "bitseq_k8":
        e = abi.env_desc(abi.BITSEQ, bs_n_bits=48, bs_k=8)
        t = abi.train_desc(abi.BITSEQ, batch=128, objective="tb", seed=6)
    elif name == "bitseq_ar_k6":
        e = abi.env_desc(abi.BITSEQ, bs_n_bits=24, bs_k=6, bs_scheme=1)
        t = abi.train_desc(abi.BITSEQ, batch=128, objective="tb", seed=6)
    elif name == "bitseq_ar_k8":
        e = abi.env_desc(abi.BITSEQ, bs_n_bits=48, bs_k=8, bs_scheme=1)
        t = abi.train_desc(abi.BITSEQ, batch=128, objective="tb", seed=6)
    elif name == "ising":
        e = abi.env_desc(abi.ISING, is_side=4, is_sigma=0.2)
        t = abi.train_desc(abi.ISING, batch=128, objective="tb", seed=7, hidden=(256, 256))
    else:
        raise KeyError(name)
    if check:
        t.precision = abi.PREC_FP64_CHECK
    return e, t


def _terminals(tr, it=0, eps=1.0):
    """Terminal states of a device forward rollout (a valid terminal of every trajectory)."""
    tr.forward_rollout(it, eps)
    return tr.batch(("terminal_state",))["terminal_state"].copy()


REF_CASES = [("hypergrid", True), ("hypergrid", False), ("hypergrid_db", False), ("dag_mdb", True),
             ("dag_mdb", False), ("bitseq_k6", True), ("bitseq_ar_k6", True), ("ising", True), ("ising", False)]


@pytest.mark.parametrize("name,check", REF_CASES)
def test_backward_rollout_bitexact_vs_reference(name, check):
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = _cfg(name, check)
    tr = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    ref.set_params(*tr.params())
    terms = _terminals(tr, it=2)
    key = (0x1234ABCD, 0x9E3779B97F4A7C15)
    tr.backward_rollout(terms, key)
    ref.backward_rollout(terms, key)
    bd, br = tr.batch(), ref.batch(tr.T)
    for k in REF_FIELDS + (("delta",) if name == "dag_mdb" else ()):
        assert np.array_equal(bd[k], br[k]), (name, k)
    assert np.array_equal(bd["terminal_state"], terms)
    ld, lr = tr.compute_grads(), ref.compute_grads()
    if check:
        assert abs(ld - lr) <= 1e-9 * max(1.0, abs(lr)), (ld, lr)
        gd, gr = tr.grads()[0], ref.grads()[0]
        assert np.max(np.abs(gd - gr)) <= 1e-9 * max(1.0, np.max(np.abs(gr)))
    else:
        assert abs(ld - lr) <= 1e-4 * max(1.0, abs(lr)), (ld, lr)
    tr.close()


@pytest.mark.parametrize("name", ["bitseq_k8", "bitseq_ar_k8"])
def test_backward_rollout_bitseq_k8_matches_check_mode(name):
    e, t = _cfg(name, False)
    e2, t2 = _cfg(name, True)
    fast, chk = engine.Trainer(e, t), engine.Trainer(e2, t2)
    chk.set_params(*fast.params())
    terms = _terminals(fast)
    key = (7, 11)
    fast.backward_rollout(terms, key)
    chk.backward_rollout(terms, key)
    bf, bc = fast.batch(), chk.batch()
    for k in FIELDS:
        assert np.array_equal(bf[k], bc[k]), k
    lf, lc = fast.compute_grads(), chk.compute_grads()
    assert abs(lf - lc) <= 1e-3 * max(1.0, abs(lc)), (lf, lc)
    fast.close()
    chk.close()


@pytest.mark.parametrize("name,check", [("hypergrid", False), ("dag_mdb", True), ("ising", False),
                                        ("bitseq_k6", True)])
def test_rollout_from_actions_replays_reference_batch(name, check):
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = _cfg(name, check)
    tr = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    ref.rollout(5, 0.5)
    br = ref.batch(tr.T)
    acts = np.where(np.arange(tr.T)[None, :] < br["lengths"][:, None], br["fwd_actions"], -1)
    tr.rollout_from_actions(acts)
    bd = tr.batch()
    for k in REF_FIELDS:
        assert np.array_equal(bd[k], br[k]), (name, k)
    tr.close()


def test_rollout_from_actions_rejects_illegal():
    e, t = _cfg("hypergrid", False)
    tr = engine.Trainer(e, t)
    acts = np.full((tr.local_batch, tr.T), -1, dtype=np.int32)  # never terminates
    with pytest.raises(engine.contract_violation):
        tr.rollout_from_actions(acts)
    acts[:, 0] = 99
    with pytest.raises(engine.contract_violation):
        tr.rollout_from_actions(acts)
    tr.close()


@pytest.mark.parametrize("name,check,tol", [("hypergrid", True, 1e-9), ("dag_mdb", True, 1e-9),
                                            ("bitseq_k6", True, 1e-9), ("bitseq_ar_k6", True, 1e-9),
                                            ("ising", True, 1e-9),
                                            ("ising", False, 5e-2)])
def test_mc_terminal_logprob_all_envs(name, check, tol):
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e, t = _cfg(name, check)
    tr = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    tr.forward_rollout(0, 0.0)
    tr.train_step(1e-3)  # a non-initial policy
    ref.set_params(*tr.params())
    terms = _terminals(tr, it=3)[:40]
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 2**63, size=(len(terms), 2), dtype=np.uint64)
    K = 5
    dev = tr.mc_terminal_logprob(terms, keys, K)
    want = np.array([ref.mc_logprob(terms[i], keys[i], K) for i in range(len(terms))])
    err = np.max(np.abs(dev - want))
    print(f"{name} check={check}: max |device - reference| = {err:.2e}")
    assert np.all(np.isfinite(dev)) and err <= tol * max(1.0, np.max(np.abs(want))), (dev, want)
    tr.close()


def test_pearson_bitseq_k8_bf16_vs_check_mode():
    """The device `pearson` metric on the bf16 k = 8 lockstep path (n = 48: 6 slots, 2880 test
    strings x 10 walks) against the fp64 check mode on the same parameters."""
    e, t = _cfg("bitseq_k8", False)
    e2, t2 = _cfg("bitseq_k8", True)
    fast, chk = engine.Trainer(e, t), engine.Trainer(e2, t2)
    fast.run(0, 30)
    chk.set_params(*fast.params())
    pf, pc = fast.pearson(30, 10), chk.pearson(30, 10)
    print(f"pearson bf16 {pf:.5f} fp64 {pc:.5f}")
    assert -1.0 <= pf <= 1.0 and abs(pf - pc) <= 2e-2, (pf, pc)
    fast.close()
    chk.close()


@pytest.mark.parametrize("name,batch", [("ising", 40), ("bitseq_k8", 200)])
def test_lockstep_ragged_batch(name, batch):
    """The lockstep (bitseq / Ising) bf16 path at a batch that is not a multiple of 128 (pad
    rows fill the last 128-row tile and carry no loss): eps = 1 trajectories bit-exact with the
    oracle, loss / gradient against the fp64 check mode on the same batch."""
    e, t = _cfg(name, False)
    t.batch_size = batch
    e2, t2 = _cfg(name, True)
    t2.batch_size = batch
    d, chk = engine.Trainer(e, t), engine.Trainer(e2, t2)
    o = O.Oracle(e, t)
    d.forward_rollout(3, 1.0)
    o.rollout_uniform(3)
    bd, bo = d.batch(), o.batch()
    for k in FIELDS:
        assert np.array_equal(bd[k], bo[k]), k
    chk.set_params(*d.params())
    acts = np.where(np.arange(d.T)[None, :] < bd["lengths"][:, None], bd["fwd_actions"], -1)
    chk.rollout_from_actions(acts)
    ld, lc = d.compute_grads(), chk.compute_grads()
    gd, gc = d.grads()[0], chk.grads()[0]
    rel = np.linalg.norm(gd - gc) / np.linalg.norm(gc)
    print(f"{name} B={batch}: loss {ld:.6f} vs {lc:.6f}, grad rel-L2 {rel:.2e}")
    assert abs(ld - lc) <= 1e-4 * max(1.0, abs(lc)) and rel < 5e-2, (ld, lc, rel)
    d.close()
    chk.close()


@pytest.mark.parametrize("name", ["ising", "bitseq_k8"])
@pytest.mark.parametrize("objective", ["db", "subtb"])
def test_lockstep_flow_objectives_vs_check_mode(name, objective):
    """DB and SubTB on the lockstep bitseq / Ising bf16 path (the log-flow head rides as head
    column A; k_ls_loss_flow): loss and gradients on the same batch against the fp64 check
    mode (the reference's operation order), with the lockstep bf16 tolerances of DESIGN §2."""
    e, t = _cfg(name, False)
    t.objective = abi.OBJECTIVES[objective]
    e2, t2 = _cfg(name, True)
    t2.objective = abi.OBJECTIVES[objective]
    d, chk = engine.Trainer(e, t), engine.Trainer(e2, t2)
    d.run(0, 3)  # a policy with a non-trivial flow head
    chk.set_params(*d.params())
    d.forward_rollout(3, 0.0)
    bd = d.batch()
    acts = np.where(np.arange(d.T)[None, :] < bd["lengths"][:, None], bd["fwd_actions"], -1)
    chk.rollout_from_actions(acts)
    ld, lc = d.compute_grads(), chk.compute_grads()
    gd, gc = d.grads()[0], chk.grads()[0]
    rel = np.linalg.norm(gd - gc) / np.linalg.norm(gc)
    off_flw = len(gc) - 257  # flow head [H][1] + bias, the last parameters
    relf = np.linalg.norm(gd[off_flw:] - gc[off_flw:]) / max(np.linalg.norm(gc[off_flw:]), 1e-30)
    print(f"{name} {objective}: loss {ld:.6f} vs {lc:.6f}, grad rel-L2 {rel:.2e}, flow head {relf:.2e}")
    assert abs(ld - lc) <= 1e-3 * max(1.0, abs(lc)), (ld, lc)
    # the whole-gradient bound here is loose (bf16 floor: the per-tensor bounds against the
    # bf16 operand model are in test_device_parity.py); the flow head must be tight
    assert rel < 2e-1 and relf < 5e-2, (rel, relf)
    d.close()
    chk.close()
