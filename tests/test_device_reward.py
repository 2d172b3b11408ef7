"""GPU: the batched terminal-reward kernels (csrc/reward.cu) against the oracle, bit for bit.

Random terminal states of every env are packed like the device batch (envs.cuh pack), scored
by gfnx_log_rewards, and compared with the restatement's log_reward_of on the same packed
words (bit-exact: the fp64 additions follow the reference's order). The device-pointer entry
(word-major SoA, the layout the B sweep of bench.py streams) must equal the host entry at a
size-independent level: 2^20 states, every value identical.
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu


def random_terminals(e, t, n, rng):
    """[n, SW] uint32 packed terminal states of env e (envs.cuh pack layouts)."""
    sh = engine.env_shape(e)
    SW = sh.state_words
    w = np.zeros((n, SW), dtype=np.uint32)
    if e.kind == abi.HYPERGRID:
        c = rng.integers(0, e.hg_side, size=(n, e.hg_dim)).astype(np.uint64)
        packed = np.zeros(n, dtype=np.uint64)
        for i in range(e.hg_dim):
            packed |= c[:, i] << np.uint64(8 * i)
        w[:, 0] = (packed & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        if SW > 1:
            w[:, 1] = (packed >> np.uint64(32)).astype(np.uint32)
    elif e.kind == abi.BITSEQ:
        slots = e.bs_n_bits // e.bs_k
        tok = rng.integers(0, 1 << e.bs_k, size=(n, slots)).astype(np.uint32)
        tw = (slots + 3) // 4
        for i in range(slots):
            w[:, i // 4] |= tok[:, i] << np.uint32(8 * (i % 4))
        w[:, tw] = np.uint32((1 << slots) - 1 if slots < 32 else 0xFFFFFFFF)
    elif e.kind == abi.ISING:
        D = e.is_side * e.is_side
        nw = SW // 2
        for k in range(nw):
            bits = min(32, D - 32 * k)
            full = np.uint32(0xFFFFFFFF if bits == 32 else (1 << bits) - 1)
            w[:, k] = full
            w[:, nw + k] = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32) & full
    else:  # DAG: random acyclic graph (edges from lower to higher rank under a permutation)
        d = e.dag_d
        for i in range(n):
            perm = rng.permutation(d)
            rows = [0] * d
            for a in range(d):
                for b in range(a + 1, d):
                    if rng.random() < 0.4:
                        rows[perm[a]] |= 1 << int(perm[b])
            for u in range(d):
                w[i, u >> 1] |= np.uint32(rows[u] << (16 * (u & 1)))
    return w


ENVS = [
    ("hypergrid_20x4", lambda: abi.config("hypergrid_tb_b16")),
    ("bitseq_n120_k8", lambda: (abi.env_desc(abi.BITSEQ, bs_n_bits=120, bs_k=8), abi.train_desc(abi.BITSEQ, batch=128))),
    ("bitseq_n48_k8", lambda: (abi.env_desc(abi.BITSEQ, bs_n_bits=48, bs_k=8), abi.train_desc(abi.BITSEQ, batch=128))),
    ("ising_10x10", lambda: (abi.env_desc(abi.ISING, is_side=10, is_sigma=0.2), abi.train_desc(abi.ISING, batch=128))),
    ("ising_6x6", lambda: (abi.env_desc(abi.ISING, is_side=6, is_sigma=0.2), abi.train_desc(abi.ISING, batch=128))),
    ("dag_d5_bge", lambda: abi.config("dag_mdb_b8192")),
]


@pytest.mark.parametrize("name,mk", ENVS)
def test_log_rewards_bitexact_vs_oracle(name, mk):
    e, t = mk()
    rng = np.random.default_rng(7)
    st = random_terminals(e, t, 3000, rng)
    d = engine.Trainer(e, t)
    o = O.Oracle(e, t)
    want = np.array([o.log_reward_of_state(s) for s in st])
    for n in (3000, 2999):  # vectorised kernels (n % 8 == 0) and the scalar tails
        got = d.log_rewards(st[:n])
        assert np.array_equal(got, want[:n]), (n, np.abs(got - want[:n]).max())
    d.close()


@pytest.mark.parametrize("name,mk", [ENVS[1], ENVS[3]])
def test_log_rewards_reject_non_terminal_states(name, mk):
    e, t = mk()
    st = random_terminals(e, t, 64, np.random.default_rng(1))
    st[5, 0 if e.kind == abi.ISING else -1] &= np.uint32(0xFFFFFFFE)  # one site / slot unassigned
    d = engine.Trainer(e, t)
    with pytest.raises(engine.contract_violation):
        d.log_rewards(st)
    d.close()


@pytest.mark.parametrize("name,mk", ENVS)
def test_device_soa_entry_equals_host_entry_at_sweep_size(name, mk):
    import torch
    e, t = mk()
    n = 1 << 20
    st = random_terminals(e, t, n if e.kind != abi.DAG else 4096, np.random.default_rng(3))
    if e.kind == abi.DAG:  # tile the (slow to generate) DAG states
        st = np.tile(st, (n // len(st), 1))
    d = engine.Trainer(e, t)
    want = d.log_rewards(st)
    soa = torch.from_numpy(np.ascontiguousarray(st.T).view(np.int32)).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    d.log_rewards_device(soa.data_ptr(), n, out.data_ptr())
    d.synchronize()
    assert np.array_equal(out.cpu().numpy(), want)
    d.close()
