"""CPU, world_size 2 over gloo: the data-parallel sharding the device engine uses.

Rank r owns trajectories [r*B/2, (r+1)*B/2) and draws them with GLOBAL indices
(fold_in(step_key, b), env_core.hpp:268), so shards reproduce the full batch exactly.
Losses are normalised by GLOBAL counts (B for TB/SubTB, all-reduced n_steps for DB
objectives.cpp:112-113, n for MDB :224); summing the shards' gradients (the NCCL
all-reduce on the GPU) must give the full-batch gradient.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_16592_b200 import abi

CASES = [("hypergrid_tb_b16", abi.TB), ("hypergrid_tb_b16", abi.DB), ("hypergrid_tb_b16", abi.SUBTB),
         ("dag_mdb_b8192", abi.MDB)]


def _worker(rank, world, port, name, obj, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    e, t = abi.config(name, batch=16, objective=obj)
    B = t.batch_size
    b0, b1 = B * rank // world, B * (rank + 1) // world
    o = O.Oracle(e, t, b0=b0, nb=b1 - b0)
    o.rollout(0, o.schedule("explore", 0))
    n_steps, n_mdb = o.counts()
    cnt = torch.tensor([n_steps, n_mdb], dtype=torch.float64)
    dist.all_reduce(cnt)
    norm = {abi.DB: cnt[0].item(), abi.MDB: cnt[1].item()}.get(obj, float(B))
    loss = o.compute_grads(norm)
    g, dz = o.grads()
    buf = torch.from_numpy(np.concatenate([g, [dz, loss]]))
    dist.all_reduce(buf)
    if rank == 0:
        q.put((buf.numpy().copy(), o.batch()["fwd_actions"].copy()))
    else:
        q.put(None)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,obj", CASES)
def test_two_rank_shards_equal_full_batch(name, obj, oracle_built):
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + obj
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, obj, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    reduced, acts0 = next(r for r in res if r is not None)
    e, t = abi.config(name, batch=16, objective=obj)
    full = O.Oracle(e, t)
    full.rollout(0, full.schedule("explore", 0))
    assert np.array_equal(full.batch()["fwd_actions"][:8], acts0)  # global-index RNG
    loss = full.compute_grads()
    g, dz = full.grads()
    n = g.size
    assert np.allclose(reduced[:n], g, rtol=1e-10, atol=1e-13 * np.abs(g).max())
    assert np.isclose(reduced[n], dz, rtol=1e-10, atol=1e-14)
    assert np.isclose(reduced[n + 1], loss, rtol=1e-12)
