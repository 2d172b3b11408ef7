"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref/libgfnref.so).

Run here (where /root/reference exists and oracle/Makefile built _ref):
    python tests/golden/make_golden.py
Writes tests/golden/*.json. Floats are stored as C99 hex strings (bit-exact).
The cases are small (B <= 32) so the fixtures stay tiny; they pin the oracle
restatement and the device check mode without the reference on the GPU box.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2511_16592_b200 import abi  # noqa: E402
from oracle.oracle import RefLib, fold_in, make_key  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def hx(v):
    return float(v).hex()


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


CASES = {
    # BASELINE config #1 (hypergrid 20^4, TB, B=16, 2x256) and the SURVEY A.3 hand-offs
    "hypergrid_tb_b16": (abi.env_desc(abi.HYPERGRID, hg_dim=4, hg_side=20),
                         abi.train_desc(abi.HYPERGRID, batch=16, objective="tb"), 4),
    "hypergrid_db_b16": (abi.env_desc(abi.HYPERGRID, hg_dim=4, hg_side=20),
                         abi.train_desc(abi.HYPERGRID, batch=16, objective="db"), 3),
    "hypergrid_subtb_b16": (abi.env_desc(abi.HYPERGRID, hg_dim=4, hg_side=20),
                            abi.train_desc(abi.HYPERGRID, batch=16, objective="subtb"), 3),
    "hypergrid_mdb_d2": (abi.env_desc(abi.HYPERGRID, hg_dim=2, hg_side=8),
                         abi.train_desc(abi.HYPERGRID, batch=16, objective="mdb"), 3),
    "bitseq_k6_tb_b16": (abi.env_desc(abi.BITSEQ, bs_n_bits=120, bs_k=6),
                         abi.train_desc(abi.BITSEQ, batch=16, objective="tb"), 2),
    "bitseq_n8k2_db_b16": (abi.env_desc(abi.BITSEQ, bs_n_bits=8, bs_k=2),
                           abi.train_desc(abi.BITSEQ, batch=16, objective="db"), 3),
    # the autoregressive-fixed scheme (SeqScheme::kAutoregressiveFixed, sequences.cpp:236-352)
    "bitseq_ar_k6_tb_b16": (abi.env_desc(abi.BITSEQ, bs_n_bits=120, bs_k=6, bs_scheme=1),
                            abi.train_desc(abi.BITSEQ, batch=16, objective="tb"), 2),
    "bitseq_ar_n16k4_subtb_b16": (abi.env_desc(abi.BITSEQ, bs_n_bits=16, bs_k=4, bs_scheme=1),
                                  abi.train_desc(abi.BITSEQ, batch=16, objective="subtb"), 3),
    "ising_n10_tb_b8": (abi.env_desc(abi.ISING, is_side=10, is_sigma=0.2),
                        abi.train_desc(abi.ISING, batch=8, objective="tb"), 2),
    "ising_n3_subtb_b16": (abi.env_desc(abi.ISING, is_side=3, is_sigma=0.2),
                           abi.train_desc(abi.ISING, batch=16, objective="subtb", hidden=(64, 64)), 3),
    "dag_bge_mdb_b32": (abi.env_desc(abi.DAG, dag_d=5, dag_score=abi.BGE),
                        abi.train_desc(abi.DAG, batch=32, objective="mdb"), 3),
    "dag_lingauss_db_b32": (abi.env_desc(abi.DAG, dag_d=4, dag_score=abi.LINGAUSS),
                            abi.train_desc(abi.DAG, batch=32, objective="db", eps=0.3), 3),
}


def struct_dict(s):
    out = {}
    for name, _ in s._fields_:
        v = getattr(s, name)
        if hasattr(v, "_fields_"):
            v = struct_dict(v)
        elif hasattr(v, "__len__") and not isinstance(v, (bytes, str)):
            v = list(v)
        elif isinstance(v, float):
            v = hx(v)
        out[name] = v
    return out


def make(name, env, train, iters):
    from paper_2511_16592_b200 import engine  # only for env_shape (host-side, no GPU)
    T = engine.env_shape(env).max_traj_len
    r = RefLib(env, train)
    p0, z0 = r.params()
    rec = dict(name=name, env=struct_dict(env), train=struct_dict(train), T=T,
               init_params_digest=digest(p0), init_params_head=[hx(v) for v in p0[:4]],
               init_params_tail=[hx(v) for v in p0[-4:]], iterations=[])
    for it in range(iters):
        lr = float(np.float64(train.lr.start_value))
        from oracle.oracle import Oracle  # schedule helper
        o = Oracle(env, train)
        eps = o.schedule("explore", it)
        lr = o.schedule("lr", it)
        r.rollout(it, eps)
        b = r.batch(T)
        loss = r.compute_grads()
        g, dz = r.grads()
        r.apply_adam(lr)
        p, z = r.params()
        rec["iterations"].append(dict(
            it=it, eps=hx(eps), lr=hx(lr),
            lengths=b["lengths"].tolist(),
            fwd_actions=b["fwd_actions"].tolist(),
            log_rewards=[hx(v) for v in b["log_rewards"]],
            log_pb_digest=digest(b["log_pb"]), delta_digest=digest(b["delta"]),
            terminal_keys=b["terminal_keys"],
            loss=hx(loss), dlogz=hx(dz), grad_digest=digest(g),
            grad_head=[hx(v) for v in g[:4]], grad_absmax=hx(np.abs(g).max()),
            params_digest=digest(p), log_z=hx(z)))
    with open(os.path.join(HERE, name + ".json"), "w") as f:
        json.dump(rec, f, indent=0)
    return rec


def main():
    for name, (e, t, iters) in CASES.items():
        make(name, e, t, iters)
        print("wrote", name)
    # RNG known answers (rng.cpp:19-39)
    from oracle.oracle import ref_lib
    import ctypes as C
    L = ref_lib("port")
    kat = []
    for (hi, lo, c0, c1) in [(0, 0, 0, 0), (2**64 - 1, 2**64 - 1, 2**64 - 1, 2**64 - 1),
                             (0xa4093822299f31d0, 0x082efa98ec4e6c89, 0x243f6a8885a308d3, 0x13198a2e03707344),
                             (0x9E3779B97F4A7C15, 0, 1000, 0x3C6EF372FE94F82B)]:
        out = (C.c_uint64 * 2)()
        L.ref_threefry(hi, lo, c0, c1, out)
        kat.append(dict(key=[hex(hi), hex(lo)], ctr=[hex(c0), hex(c1)], out=[hex(out[0]), hex(out[1])]))
    k = fold_in(fold_in(make_key(0), 1000), 0)
    uni = [dict(idx=i, u=hx(L.ref_uniform_fold(k[0], k[1], i))) for i in range(64)]
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump(dict(threefry=kat, uniform_key=[hex(k[0]), hex(k[1])], uniform=uni), f, indent=0)
    print("wrote rng")


if __name__ == "__main__":
    main()
