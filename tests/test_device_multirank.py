"""GPU: libgfnx's world > 1 path, run as two ranks on ONE GPU (in-process group).

Each rank is a gfnx_ctx in the same gfnx_group, driven by its own host thread; the group's
all-reduce (libgfnx's peer-memory sum kernel, csrc/group.cu) replaces NCCL. The data-parallel
contract of SURVEY §8(e):
* rank r simulates the global trajectories [r B / W, (r + 1) B / W) with the reference RNG
  stream indexed by the GLOBAL trajectory index (env_core.hpp:268), so the ranks' batches
  concatenate to the world = 1 batch bit for bit;
* the DB / MDB normalisers are the all-reduced global counts (objectives.cpp:112-113,224), TB /
  SubTB use the global B, so the summed gradient equals the full-batch gradient (fp32
  summation order aside) and is identical on every rank;
* replicated Adam keeps the ranks' parameters identical.
"""
import threading

import numpy as np
import pytest

from paper_2511_16592_b200 import abi, engine

pytestmark = pytest.mark.gpu


def _on_ranks(trainers, fn):
    """fn(rank, trainer) on one thread per rank (a collective needs every rank)."""
    out, errs = [None] * len(trainers), []

    def work(r):
        try:
            out[r] = fn(r, trainers[r])
        except BaseException as ex:  # noqa: BLE001 - re-raised below
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(len(trainers))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


CASES = [
    ("hypergrid_db_b65536", dict(batch=3000), "bf16"),
    ("hypergrid_db_b65536", dict(batch=2048, objective="tb"), "bf16"),
    ("hypergrid_subtb_b65536", dict(batch=1000), "bf16"),
    ("hypergrid_db_b65536", dict(batch=1500, objective="mdb"), "bf16"),
    ("dag_mdb_b8192", dict(batch=1024), "bf16"),
    ("hypergrid_db_b65536", dict(batch=64), "fp64"),
    ("dag_mdb_b8192", dict(batch=64), "fp64"),
]


@pytest.mark.parametrize("name,kw,prec", CASES)
def test_two_ranks_on_one_gpu_equal_the_single_rank_job(name, kw, prec):
    e, t = abi.config(name, **kw)
    if prec == "fp64":
        t.precision = abi.PREC_FP64_CHECK
    one = engine.Trainer(e, t)
    g = engine.Group(2)
    ranks = [engine.Trainer(e, t, rank=r, world=2, group=g) for r in range(2)]
    try:
        for it in range(2):
            eps = 0.5 if it == 0 else 0.0
            p0, z0 = one.params()
            st = one.adam_state()
            for tr in ranks:  # identical state on every rank (the policy decides the eps < 1 draws)
                tr.set_params(p0, z0)
                tr.set_adam_state(*st)
            one.forward_rollout(it, eps)
            l1 = one.compute_grads()
            g1, dz1 = one.grads()
            b1 = one.batch()

            def step(r, tr):
                tr.forward_rollout(it, eps)
                loss = tr.compute_grads()
                return loss, tr.grads(), tr.batch()

            res = _on_ranks(ranks, step)
            # batches: the rank slices concatenate to the single-rank batch, bit for bit
            for k in b1:
                assert np.array_equal(np.concatenate([res[0][2][k], res[1][2][k]]), b1[k]), k
            # gradients: identical on both ranks (rank-order sum), equal to the full batch
            (ga, dza), (gb, dzb) = res[0][1], res[1][1]
            assert np.array_equal(ga, gb) and dza == dzb
            tol = 1e-12 if prec == "fp64" else 2e-5
            assert np.linalg.norm(ga - g1) <= tol * np.linalg.norm(g1), np.linalg.norm(ga - g1) / np.linalg.norm(g1)
            assert abs(dza - dz1) <= tol * max(abs(dz1), 1e-30)
            # loss: all-reduced partials
            assert abs(res[0][0] - l1) <= tol * abs(l1) and res[0][0] == res[1][0]
            # one replicated Adam step from identical state keeps the ranks identical
            lr = 1e-3
            one.train_step(lr, read_loss=False)
            _on_ranks(ranks, lambda r, tr: tr.train_step(lr, read_loss=False))
            pa, za = ranks[0].params()
            pb, zb = ranks[1].params()
            assert np.array_equal(pa, pb) and za == zb
            # the step equals the single-rank step up to the gradients' summation order (Adam's
            # m / sqrt(v) can flip where a gradient component is ~0)
            p1, _ = one.params()
            assert np.linalg.norm(pa - p1) <= (1e-6 if prec == "fp64" else 2e-2) * np.linalg.norm(p1 - p0)
    finally:
        for tr in ranks:
            tr.close()
        g.close()
        one.close()


def test_group_iteration_pipeline_runs():
    """gfnx_run on both ranks (rollout, counts + gradient all-reduce, Adam) stays in lockstep."""
    e, t = abi.config("hypergrid_db_b65536", batch=4096)
    g = engine.Group(2)
    ranks = [engine.Trainer(e, t, rank=r, world=2, group=g) for r in range(2)]
    try:
        losses = _on_ranks(ranks, lambda r, tr: tr.run(0, 5, read_losses=True))
        assert np.array_equal(losses[0], losses[1]) and np.all(np.isfinite(losses[0]))
        pa, _ = ranks[0].params()
        pb, _ = ranks[1].params()
        assert np.array_equal(pa, pb)
    finally:
        for tr in ranks:
            tr.close()
        g.close()
