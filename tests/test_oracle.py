"""CPU: the oracle restatement pinned against the reference (golden fixtures + live _ref)."""
import hashlib

import numpy as np
import pytest

from golden_util import CASES, fh, load, load_rng
from oracle import oracle as O
from paper_2511_16592_b200 import abi


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def test_threefry_random123_kat(oracle_built):
    # Random123 threefry2x64-20 known answer (key 0, ctr 0) and reference-recorded vectors
    assert O.threefry((0, 0), 0, 0) == (0xc2b6e3a8c2c69865, 0x6f81ed42f350084d)
    for kat in load_rng()["threefry"]:
        key = tuple(int(x, 16) for x in kat["key"])
        ctr = tuple(int(x, 16) for x in kat["ctr"])
        assert O.threefry(key, *ctr) == tuple(int(x, 16) for x in kat["out"])


def test_uniform_fold_fixture(oracle_built):
    rng = load_rng()
    key = tuple(int(x, 16) for x in rng["uniform_key"])
    for e in rng["uniform"]:
        assert O.uniform_scalar(O.fold_in(key, e["idx"])) == fh(e["u"])
    # uniform_scalar(fold_in(fold_in(make_key(0),1000),0))
    assert O.uniform_scalar(O.fold_in(O.fold_in(O.make_key(0), 1000), 0)) == 0.44468281925543396


def test_categorical_and_eps_uniform_hand_values(oracle_built):
    # objectives test_objectives.cpp:233-263 hand values
    import ctypes as C
    L = O.lib()
    logits = np.log(np.array([0.8, 0.2]))
    mask = np.ones(2, np.uint8)
    probs = np.zeros(2)
    for eps, want in ((0.0, (0.8, 0.2)), (1.0, (0.5, 0.5)), (0.5, (0.65, 0.35))):
        n = L.orc_eps_uniform(O._p(logits), O._p(mask), 2, eps, O._p(probs))
        assert n == 2 and np.allclose(probs, want, rtol=1e-12)
    none = np.zeros(2, np.uint8)
    assert L.orc_eps_uniform(O._p(logits), O._p(none), 2, 0.1, O._p(probs)) == 0
    w = np.array([0.0, 0.0])
    key = np.array([1, 2], dtype=np.uint64)
    assert L.orc_categorical(O._p(key), O._p(w), 2) == -1


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(oracle_built, name):
    g = load(name)
    o = O.Oracle(g["env_desc"], g["train_desc"])
    p0, _ = o.params()
    assert digest(p0) == g["init_params_digest"]
    for rec in g["iterations"]:
        it = rec["it"]
        assert o.schedule("explore", it) == fh(rec["eps"])
        o.rollout(it, fh(rec["eps"]))
        b = o.batch()
        assert b["lengths"].tolist() == rec["lengths"]
        assert b["fwd_actions"].tolist() == rec["fwd_actions"]
        assert [v.hex() for v in b["log_rewards"]] == rec["log_rewards"]
        assert digest(b["log_pb"]) == rec["log_pb_digest"]
        assert digest(b["delta"]) == rec["delta_digest"]
        loss = o.compute_grads()
        gr, dz = o.grads()
        assert loss.hex() == rec["loss"]
        assert dz.hex() == rec["dlogz"]
        assert digest(gr) == rec["grad_digest"]
        o.apply_adam(fh(rec["lr"]))
        p, z = o.params()
        assert digest(p) == rec["params_digest"]
        assert z.hex() == rec["log_z"]


def test_survey_a3_hypergrid_tb_goldens(oracle_built):
    """hypergrid 20^4 TB, B=16, seed 0, iterations 0-9."""
    e, t = abi.config("hypergrid_tb_b16")
    o = O.Oracle(e, t)
    p, _ = o.params()
    assert p[0].hex() == "0x1.c3e2d54359589p-4"
    assert p[80 * 256 - 1].hex() == "-0x1.d902b717149b3p-5"
    assert p[80 * 256 + 256 + 256 * 256 + 256].hex() == "0x1.461737365dce4p-5"  # fwd_head W[0]
    losses = [o.iteration(it) for it in range(10)]
    assert losses[0] == 23.345431030553069
    want = [17.709076540981371, 12.603639958851689, 17.501225989769424, 14.949589483206834,
            16.65641260147212, 18.85392040443212, 14.396213899500065, 11.477903022286563,
            10.753945807759033]
    # A.3 was recorded with the shipped (FMA-contracting) build; floats agree to ~1 ulp
    assert np.allclose(losses[1:], want, rtol=1e-13, atol=0)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("cfg", [("hypergrid_tb_b16", 6), ("dag_mdb_b8192", 2)])
def test_oracle_matches_live_reference(oracle_built, cfg):
    name, iters = cfg
    e, t = abi.config(name, batch=64) if name.startswith("dag") else abi.config(name)
    o, r = O.Oracle(e, t), O.RefLib(e, t)
    T = o.shape.max_traj_len
    for it in range(iters):
        lo, lr_ = o.iteration(it), r.iteration(it)
        assert lo == lr_
        bo, br = o.batch(), r.batch(T)
        assert np.array_equal(bo["fwd_actions"], br["fwd_actions"])
        assert np.array_equal(o.params()[0], r.params()[0])


def test_oracle_rejects_like_reference(oracle_built):
    e = abi.env_desc(abi.HYPERGRID, hg_r0=0.0)
    with pytest.raises(ValueError, match="r0 must be positive"):
        O.Oracle(e, abi.train_desc(abi.HYPERGRID))
    e = abi.env_desc(abi.BITSEQ, bs_n_bits=12, bs_k=5)
    with pytest.raises(ValueError, match="k must divide"):
        O.Oracle(e, abi.train_desc(abi.BITSEQ))
    with pytest.raises(ValueError, match="mdb objective needs the stop action"):
        O.Oracle(abi.env_desc(abi.ISING), abi.train_desc(abi.ISING, objective="mdb"))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_reference_mc_logprob_and_pearson_shims(oracle_built):
    """The shim entry points the GPU tests use as checkers: mc_terminal_logprob of the origin
    cell has a single backward path (un-stop), so every sample equals log pi(stop | s0); the
    bitseq pearson metric is a correlation in [-1, 1]."""
    import numpy as np
    from paper_2511_16592_b200 import abi
    e = abi.env_desc(abi.HYPERGRID, hg_dim=2, hg_side=8)
    t = abi.train_desc(abi.HYPERGRID, batch=16, objective="tb", seed=1)
    ref = O.RefLib(e, t)
    lp1 = ref.mc_logprob(np.array([0], np.uint32), (1, 2), 1)
    lp8 = ref.mc_logprob(np.array([0], np.uint32), (3, 4), 8)
    assert np.isfinite(lp1) and lp1 < 0.0 and abs(lp1 - lp8) < 1e-12
    eb = abi.env_desc(abi.BITSEQ, bs_n_bits=8, bs_k=2)
    tb = abi.train_desc(abi.BITSEQ, batch=16, objective="tb", seed=3)
    r = O.RefLib(eb, tb).pearson(0)
    assert -1.0 <= r <= 1.0
