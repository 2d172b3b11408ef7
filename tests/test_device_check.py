"""GPU: the fp64 check mode of libgfnx against the oracle and the reference golden fixtures.

Check mode reproduces the reference operation order (SIMT fp64, no FMA contraction):
sampled actions, lengths, terminal states, log-rewards and log P_B are required to be
bit-exact; losses, gradients and Adam-updated parameters agree within 1e-10 relative
(device exp/log differ from glibc's by <= 1 ulp). Teacher forcing re-imports the oracle's
parameters and Adam state before every iteration.
"""
import ctypes as C

import numpy as np
import pytest

from golden_util import CASES, fh, load, load_rng
from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu


def _check_desc(t):
    t2 = abi.TrainDesc.from_buffer_copy(t)
    t2.precision = abi.PREC_FP64_CHECK
    return t2


def test_threefry_device_bitexact():
    rng = np.random.default_rng(0)
    n = 100000
    keys = rng.integers(0, 2**63, size=(n, 2), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    ctrs = rng.integers(0, 2**63, size=(n, 2), dtype=np.uint64)
    out = engine.test_threefry(keys, ctrs)
    for i in range(0, n, 997):
        assert tuple(int(x) for x in out[i]) == O.threefry(tuple(int(x) for x in keys[i]),
                                                           int(ctrs[i, 0]), int(ctrs[i, 1]))
    z = engine.test_threefry(np.zeros((1, 2), np.uint64), np.zeros((1, 2), np.uint64))
    assert (int(z[0, 0]), int(z[0, 1])) == (0xc2b6e3a8c2c69865, 0x6f81ed42f350084d)


def test_uniform_fold_device_bitexact():
    rng = load_rng()
    key = tuple(int(x, 16) for x in rng["uniform_key"])
    u = engine.test_uniform_fold(key, np.arange(64, dtype=np.uint64))
    assert [v.hex() for v in u] == [e["u"] for e in rng["uniform"]]


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", CASES)
def test_check_mode_matches_reference(name):
    g = load(name)
    e, t = g["env_desc"], _check_desc(g["train_desc"])
    o = O.Oracle(e, g["train_desc"])
    d = engine.Trainer(e, t)
    try:
        pd, zd = d.params()
        po, zo = o.params()
        assert np.array_equal(pd, po), "mlp_init must be bit-exact (host threefry)"
        for rec in g["iterations"]:
            it = rec["it"]
            eps, lr = fh(rec["eps"]), fh(rec["lr"])
            d.forward_rollout(it, eps)
            o.rollout(it, eps)
            bd, bo = d.batch(), o.batch()
            assert bd["lengths"].tolist() == rec["lengths"]
            assert bd["fwd_actions"].tolist() == rec["fwd_actions"]
            assert [v.hex() for v in bd["log_rewards"]] == rec["log_rewards"]
            for k in ("bwd_actions", "log_pb", "delta", "terminal_state"):
                assert np.array_equal(bd[k], bo[k]), k
            loss_d = d.train_step(lr)
            loss_o = o.compute_grads()
            assert abs(loss_d - loss_o) <= 1e-10 * abs(loss_o)
            gd, dzd = d.grads()
            go, dzo = o.grads()
            assert _rel(gd, go) < 1e-9, _rel(gd, go)
            assert abs(dzd - dzo) <= 1e-9 * max(abs(dzo), 1e-300)
            o.apply_adam(lr)
            pd, zd = d.params()
            po, zo = o.params()
            assert np.abs(pd - po).max() < 1e-12
            assert abs(zd - zo) < 1e-12
            # teacher forcing: continue from the oracle's exact state
            d.set_params(po, zo)
            d.set_adam_state(*o.adam())
    finally:
        d.close()


def test_check_mode_free_running_hypergrid_tb():
    """Config #1 free-running for 10 iterations (no teacher forcing): the device check mode
    keeps producing the oracle's (== reference's) actions and the SURVEY A.3 losses."""
    e, t = abi.config("hypergrid_tb_b16")
    d = engine.Trainer(e, _check_desc(t))
    o = O.Oracle(e, t)
    want = [23.345431030553069, 17.709076540981371, 12.603639958851689, 17.501225989769424,
            14.949589483206834, 16.65641260147212, 18.85392040443212, 14.396213899500065,
            11.477903022286563, 10.753945807759033]
    for it in range(10):
        ld = d.iteration(it)
        lo = o.iteration(it)
        assert np.array_equal(d.batch()["fwd_actions"], o.batch()["fwd_actions"])
        assert abs(ld - lo) <= 1e-9 * abs(lo)
        assert abs(ld - want[it]) <= 1e-9 * want[it]
    d.close()


def test_device_errors_are_raised():
    e, t = abi.config("hypergrid_tb_b16")
    d = engine.Trainer(e, _check_desc(t))
    with pytest.raises(engine.contract_violation):
        d.train_step(1e-3)  # no batch yet
    with pytest.raises(engine.config_error):
        d.forward_rollout(0, 1.5)
    d.close()
    with pytest.raises(engine.config_error):
        engine.Trainer(abi.env_desc(abi.HYPERGRID, hg_r0=0.0), t)
