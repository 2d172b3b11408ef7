"""GPU: the device Monte-Carlo terminal log-probability (gfnx_mc_terminal_logprob, SURVEY §8(f)
rank 2) against the reference's mc_terminal_logprob (exact.hpp:229-241: backward_rollout with
the uniform backward policy, env_core.hpp:314-370, + score_trajectories, objectives.cpp:294-316)
run by oracle/_ref on the same parameters and keys — the backward paths are drawn from the same
Threefry stream, so the only difference is the bf16 policy — and, as the reference's acceptance
criterion 4 does (acceptance.cpp:314-333), the estimator against the exact terminal marginal."""
import numpy as np
import pytest

from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu

D, H = 2, 8


def packed(cells):
    return np.array([[c0 | (c1 << 8)] for c0, c1 in cells], dtype=np.uint32)


def test_mc_logprob_matches_reference():
    from oracle import oracle as O
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    e = abi.env_desc(abi.HYPERGRID, hg_dim=D, hg_side=H)
    t = abi.train_desc(abi.HYPERGRID, batch=16, objective="tb", seed=1)
    tr = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    rng = np.random.default_rng(7)
    cells = [(0, 0), (7, 7), (3, 5), (6, 1)] + [tuple(rng.integers(0, H, 2)) for _ in range(12)]
    terms = packed(cells)
    keys = rng.integers(0, 2**63, size=(len(cells), 2), dtype=np.uint64)
    for stage in range(2):
        ref.set_params(*tr.params())
        dev = tr.mc_terminal_logprob(terms, keys, 10)
        want = np.array([ref.mc_logprob(terms[i], keys[i], 10) for i in range(len(cells))])
        assert np.all(np.isfinite(dev))
        print(f"stage {stage}: max |device - reference| = {np.max(np.abs(dev - want)):.2e}")
        assert np.max(np.abs(dev - want)) < 5e-2, (stage, dev, want)  # bf16 policy vs fp64
        tr.run(0, 300)  # a trained, non-uniform policy for the second pass
    tr.close()


def test_mc_estimator_within_three_sigma_of_exact_marginal():
    e = abi.env_desc(abi.HYPERGRID, hg_dim=D, hg_side=H)
    t = abi.train_desc(abi.HYPERGRID, batch=16, objective="tb", seed=2)
    tr = engine.Trainer(e, t)
    tr.run(0, 300)
    marg, _ = tr.exact_terminal_marginal(H ** D)  # cell index c0 + H c1
    rng = np.random.default_rng(11)
    cells = [(2, 3), (5, 5), (1, 6)]
    reps = 60
    terms = np.repeat(packed(cells), reps, axis=0)
    keys = rng.integers(0, 2**63, size=(len(terms), 2), dtype=np.uint64)
    est = np.exp(tr.mc_terminal_logprob(terms, keys, 10)).reshape(len(cells), reps)
    tr.close()
    for j, (c0, c1) in enumerate(cells):
        mean, se = est[j].mean(), est[j].std(ddof=1) / np.sqrt(reps)
        assert abs(mean - marg[c0 + H * c1]) <= 3 * se + 1e-4, (j, mean, se, marg[c0 + H * c1])


def test_mc_logprob_dag_matches_reference():
    """DAG d = 4 (linear-Gaussian score): terminals are random DAGs (edges added in a random
    topological order), packed as the device packs them (row u in half u & 1 of word u >> 1)."""
    from oracle import oracle as O
    if not O.ref_available("port"):
        pytest.skip("oracle/_ref not built")
    d = 4
    e = abi.env_desc(abi.DAG, dag_d=d, dag_score=abi.LINGAUSS)
    t = abi.train_desc(abi.DAG, batch=64, seed=5, hidden=(128, 128), objective="mdb")
    tr = engine.Trainer(e, t)
    ref = O.RefLib(e, t)
    rng = np.random.default_rng(3)
    terms = []
    for _ in range(12):
        order = rng.permutation(d)
        adj = np.zeros(d, dtype=np.uint32)
        for i in range(d):
            for j in range(i + 1, d):
                if rng.random() < 0.5:
                    adj[order[i]] |= 1 << int(order[j])
        w = np.zeros(tr.state_words, dtype=np.uint32)
        for u in range(d):
            w[u >> 1] |= np.uint32(int(adj[u]) << (16 * (u & 1)))
        terms.append(w)
    terms = np.array(terms)
    keys = rng.integers(0, 2**63, size=(len(terms), 2), dtype=np.uint64)
    for stage in range(2):
        ref.set_params(*tr.params())
        dev = tr.mc_terminal_logprob(terms, keys, 8)
        want = np.array([ref.mc_logprob(terms[i], keys[i], 8) for i in range(len(terms))])
        print(f"dag stage {stage}: max |device - reference| = {np.max(np.abs(dev - want)):.2e}")
        assert np.all(np.isfinite(dev)) and np.max(np.abs(dev - want)) < 5e-2, (stage, dev, want)
        tr.run(0, 200)
    tr.close()
