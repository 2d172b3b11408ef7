"""GPU: the on-device `tv_buffer` metric (gfnx_buffer_reset / _push / gfnx_tv_buffer) against a
restatement of the reference's FifoBuffer (buffer.hpp:13-55: fixed capacity, oldest evicted
first, fed by buffer.push_batch(batch.terminal_keys) after every iteration, train.cpp:231) and
tv_distance(buffer.empirical(), grid_exact_distribution) (metrics.cpp:35-48,
hypergrid.cpp:121-140) over the terminal states the device exported for the same iterations."""
import collections

import numpy as np
import pytest

from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu

D, H = 2, 8


def exact_probs(e):
    """grid_exact_distribution: exp(log(r0 + r1 p1 + r2 p2)) in enumeration order, normalised;
    returned in the device's cell order (coordinate 0 fastest)."""
    p = {}
    z = 0.0
    for idx in np.ndindex(*([H] * D)):  # last coordinate fastest, as the reference enumerates
        ax = np.abs(np.array(idx) / (H - 1) - 0.5)
        p1, p2 = bool(np.all(0.25 < ax)), bool(np.all((0.3 < ax) & (ax < 0.4)))
        v = float(np.exp(np.log(e.hg_r0 + e.hg_r1 * p1 + e.hg_r2 * p2)))
        z += v
        p[sum(c * H ** i for i, c in enumerate(idx))] = v
    return {k: v / z for k, v in p.items()}


def cells_of(term):
    w = term[:, 0].astype(np.int64)
    return sum(((w >> (8 * i)) & 0xFF) * H ** i for i in range(D))


class Fifo:  # buffer.hpp:13-55
    def __init__(self, cap):
        self.cap, self.ring = cap, collections.deque(maxlen=cap)

    def push_batch(self, items):
        for x in items:
            self.ring.append(int(x))

    def tv(self, exact):  # metrics.cpp:35-48
        cnt = collections.Counter(self.ring)
        n = len(self.ring)
        acc = cov = 0.0
        for k, p in exact.items():
            ph = cnt[k] / n if k in cnt else 0.0
            if k in cnt:
                cov += ph
            acc += abs(ph - p)
        return 0.5 * (acc + 1.0 - cov)


@pytest.mark.parametrize("cap", [10, 40, 200000])  # batch > capacity, wrap-around, never full
def test_tv_buffer_matches_reference_fifo(cap):
    e = abi.env_desc(abi.HYPERGRID, hg_dim=D, hg_side=H)
    t = abi.train_desc(abi.HYPERGRID, batch=16, objective="tb", seed=3, iterations=100)
    tr = engine.Trainer(e, t)
    exact = exact_probs(e)
    tr.buffer_reset(cap)
    with pytest.raises(Exception):
        tr.tv_buffer()  # empirical of an empty buffer is a contract violation
    ref = Fifo(cap)
    for it in range(12):
        tr.iteration(it)
        tr.buffer_push()
        ref.push_batch(cells_of(tr.batch(["terminal_state"])["terminal_state"]))
        n, tv = tr.tv_buffer()
        assert n == len(ref.ring)
        assert abs(tv - ref.tv(exact)) < 1e-12, (it, tv, ref.tv(exact))
    tr.close()


def test_tv_buffer_config2_grid():
    """20^4 grid (BASELINE config #2) at the reference's default capacity: a distance in [0, 1]
    that drops as the buffer fills with samples of a trained-for-a-while policy."""
    e, t = abi.config("hypergrid_db_b65536", batch=4096)
    tr = engine.Trainer(e, t)
    tr.buffer_reset(200000)
    vals = []
    for it in range(60):
        tr.iteration(it)
        tr.buffer_push()
        if it in (0, 59):
            vals.append(tr.tv_buffer())
    tr.close()
    (n0, tv0), (n1, tv1) = vals
    assert n0 == 4096 and n1 == 200000
    assert 0.0 <= tv1 <= 1.0 and 0.0 <= tv0 <= 1.0
