"""ctypes mirror of include/gfnx.h (descriptor structs, enums, per-env defaults).

The defaults reproduce the reference drivers' per-environment settings
(proj/src/train.cpp:43-62 EnvDefaults, :105-137 read_settings and the
build_* functions :353-657) so one description drives the device engine,
the CPU oracle and the reference shim alike.
"""
from __future__ import annotations

import ctypes as C

# gfnx_status
OK, ERR_CONFIG, ERR_CONTRACT, ERR_NUMERIC, ERR_CUDA, ERR_NCCL = range(6)
# gfnx_env_kind
HYPERGRID, BITSEQ, ISING, DAG = range(4)
ENV_NAMES = {HYPERGRID: "hypergrid", BITSEQ: "bitseq", ISING: "ising", DAG: "dag"}
# gfnx_objective (same numbering as gfn::Objective)
DB, TB, SUBTB, FLDB, MDB = range(5)
OBJECTIVES = {"db": DB, "tb": TB, "subtb": SUBTB, "fldb": FLDB, "mdb": MDB}
# gfnx_precision
PREC_BF16, PREC_FP64_CHECK = 0, 1
# schedule kinds
CONSTANT, LINEAR, COSINE = 0, 1, 2
LINGAUSS, BGE = 0, 1


class Schedule(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pad_", C.c_int32), ("start_value", C.c_double),
                ("end_value", C.c_double), ("warmup", C.c_int64), ("horizon", C.c_int64)]


class EnvDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("hg_dim", C.c_int32), ("hg_side", C.c_int32), ("pad0_", C.c_int32),
        ("hg_r0", C.c_double), ("hg_r1", C.c_double), ("hg_r2", C.c_double),
        ("bs_n_bits", C.c_int32), ("bs_k", C.c_int32), ("bs_beta", C.c_double),
        ("bs_num_modes", C.c_int32), ("bs_scheme", C.c_int32), ("bs_modes_seed", C.c_uint64),
        ("is_side", C.c_int32), ("pad2_", C.c_int32), ("is_sigma", C.c_double),
        ("dag_d", C.c_int32), ("dag_score", C.c_int32),
        ("dag_alpha_mu", C.c_double), ("dag_alpha_w", C.c_double),
        ("dag_noise_var", C.c_double), ("dag_weight_var", C.c_double),
        ("dag_expected_in_degree", C.c_double),
        ("dag_data_n", C.c_int32), ("pad3_", C.c_int32), ("dag_data_seed", C.c_uint64),
    ]


class TrainDesc(C.Structure):
    _fields_ = [
        ("objective", C.c_int32), ("learned_backward", C.c_int32),
        ("subtb_lambda", C.c_double), ("terminal_penalty", C.c_double),
        ("batch_size", C.c_int32), ("num_hidden", C.c_int32), ("hidden", C.c_int32 * 8),
        ("logz_init", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double), ("adam_eps", C.c_double),
        ("weight_decay", C.c_double), ("z_lr", C.c_double),
        ("lr", Schedule), ("explore", Schedule),
        ("iterations", C.c_int64), ("seed", C.c_uint64),
        ("precision", C.c_int32), ("deterministic", C.c_int32),
    ]


class EnvShape(C.Structure):
    _fields_ = [("num_actions", C.c_int32), ("num_backward_actions", C.c_int32),
                ("obs_dim", C.c_int32), ("max_traj_len", C.c_int32),
                ("stop_action", C.c_int32), ("state_words", C.c_int32)]


class HostBatch(C.Structure):
    _fields_ = [("lengths", C.POINTER(C.c_int32)), ("fwd_actions", C.POINTER(C.c_int32)),
                ("bwd_actions", C.POINTER(C.c_int32)), ("log_rewards", C.POINTER(C.c_double)),
                ("log_pb", C.POINTER(C.c_double)), ("delta_log_reward", C.POINTER(C.c_double)),
                ("terminal_state", C.POINTER(C.c_uint32))]


class EbDesc(C.Structure):  # gfnx_eb_desc
    _fields_ = [("data_samples", C.c_int32), ("k", C.c_int32), ("gibbs_burn_in", C.c_int64),
                ("gibbs_thinning", C.c_int64), ("gibbs_chains", C.c_int32), ("data_batch", C.c_int32),
                ("gibbs_hottest_beta", C.c_double), ("alpha", C.c_double), ("coupling_lr", C.c_double),
                ("coupling_lr_end", C.c_double)]


class SlotView(C.Structure):
    _fields_ = [("it", C.c_int64), ("loss", C.c_double), ("n", C.c_int32),
                ("state_words", C.c_int32), ("lengths", C.POINTER(C.c_int32)),
                ("log_rewards", C.POINTER(C.c_double)), ("terminal_state", C.POINTER(C.c_uint32))]


def env_desc(kind: int, **kw) -> EnvDesc:
    """Defaults of the reference builders (train.cpp:361-366, 388-396, 637-640, 531-583)."""
    e = EnvDesc()
    e.kind = kind
    e.hg_dim, e.hg_side, e.hg_r0, e.hg_r1, e.hg_r2 = 2, 8, 1e-3, 0.5, 2.0
    e.bs_n_bits, e.bs_k, e.bs_beta, e.bs_num_modes, e.bs_modes_seed = 8, 2, 3.0, 60, 0
    e.is_side, e.is_sigma = 3, 0.2
    e.dag_d, e.dag_score = 5, LINGAUSS
    e.dag_alpha_mu, e.dag_alpha_w = 1.0, 0.0
    e.dag_noise_var, e.dag_weight_var = 0.1, 1.0
    e.dag_expected_in_degree, e.dag_data_n, e.dag_data_seed = 1.0, 100, 0
    for k, v in kw.items():
        if not hasattr(e, k):
            raise KeyError(k)
        setattr(e, k, v)
    return e


def _sched(kind, start, end, warmup=0, horizon=0) -> Schedule:
    s = Schedule()
    s.kind, s.start_value, s.end_value, s.warmup, s.horizon = kind, start, end, warmup, horizon
    return s


def train_desc(kind: int, **kw) -> TrainDesc:
    """EnvDefaults + read_settings for env `kind` (train.cpp:43-62, 105-137).

    Keyword overrides: any TrainDesc field, plus `hidden=(...)`, `objective="tb"`,
    `lr=<float>` (constant schedule), `eps=<float>` (constant exploration).
    """
    d = dict(iterations=1000, batch=16, lr=1e-3, z_lr=0.1, wd=0.0, hidden=(256, 256),
             objective="tb", eps_start=0.0, eps_end=0.0, eps_horizon=0)
    if kind == HYPERGRID:      # train.cpp:353-358
        d.update(iterations=62500)
    elif kind == BITSEQ:       # train.cpp:381-389
        d.update(iterations=50000, z_lr=0.05, wd=1e-5, eps_start=1e-3, eps_end=1e-3)
    elif kind == DAG:          # train.cpp:523-533
        d.update(iterations=100000, batch=128, lr=1e-4, hidden=(128, 128), objective="mdb",
                 eps_start=1.0, eps_end=0.1, eps_horizon=-1)
    elif kind == ISING:        # train.cpp:637-645
        d.update(iterations=20000, batch=256, hidden=(256, 256, 256, 256))
    t = TrainDesc()
    t.objective = OBJECTIVES[d["objective"]]
    t.learned_backward = 0
    t.subtb_lambda = 0.9
    t.terminal_penalty = 1.0
    t.batch_size = d["batch"]
    t.logz_init = 0.0
    t.beta1, t.beta2, t.adam_eps, t.weight_decay = 0.9, 0.999, 1e-8, d["wd"]
    t.z_lr = d["z_lr"]
    t.lr = _sched(CONSTANT, d["lr"], d["lr"], 0, 0)
    same = d["eps_start"] == d["eps_end"]
    t.explore = _sched(CONSTANT if same else LINEAR, d["eps_start"], d["eps_end"], 0,
                       d["eps_horizon"])
    t.iterations = d["iterations"]
    t.seed = 0
    t.precision = PREC_BF16
    hidden = tuple(d["hidden"])
    for k, v in kw.items():
        if k == "hidden":
            hidden = tuple(v)
        elif k == "objective":
            t.objective = OBJECTIVES[v] if isinstance(v, str) else int(v)
        elif k == "lr":
            t.lr = _sched(CONSTANT, v, v, 0, 0)
        elif k == "eps":
            t.explore = _sched(CONSTANT, v, v, 0, 0)
        elif k == "batch":
            t.batch_size = v
        elif hasattr(t, k):
            setattr(t, k, v)
        else:
            raise KeyError(k)
    t.num_hidden = len(hidden)
    for i, h in enumerate(hidden):
        t.hidden[i] = h
    return t


# BASELINE.json configs as (env_desc, train_desc) factories.
def config(name: str, **kw):
    if name == "hypergrid_tb_b16":        # config #1
        e = env_desc(HYPERGRID, hg_dim=4, hg_side=20)
        t = train_desc(HYPERGRID, batch=16, objective="tb")
    elif name in ("hypergrid_db_b65536", "hypergrid_subtb_b65536"):  # config #2
        e = env_desc(HYPERGRID, hg_dim=4, hg_side=20)
        t = train_desc(HYPERGRID, batch=65536, objective=name.split("_")[1])
    elif name == "bitseq_tb_b16384":      # config #3 (k=8 NAR; reference caps k at 6)
        e = env_desc(BITSEQ, bs_n_bits=120, bs_k=8)
        t = train_desc(BITSEQ, batch=16384, objective="tb")
    elif name == "bitseq_ar_tb_b16384":   # config #3 as written: k=8 autoregressive (fixed length)
        e = env_desc(BITSEQ, bs_n_bits=120, bs_k=8, bs_scheme=1)
        t = train_desc(BITSEQ, batch=16384, objective="tb")
    elif name == "ising_tb_b32768":       # config #4
        e = env_desc(ISING, is_side=10, is_sigma=0.2)
        t = train_desc(ISING, batch=32768, objective="tb")
    elif name == "dag_mdb_b8192":         # config #5
        e = env_desc(DAG, dag_d=5, dag_score=BGE)
        t = train_desc(DAG, batch=8192, objective="mdb")
    else:
        raise KeyError(name)
    for k, v in kw.items():
        if hasattr(e, k):
            setattr(e, k, v)
        elif k == "batch":
            t.batch_size = v
        elif k == "objective":
            t.objective = OBJECTIVES[v] if isinstance(v, str) else int(v)
        elif k == "hidden":
            t.num_hidden = len(v)
            for i, h in enumerate(v):
                t.hidden[i] = h
        else:
            setattr(t, k, v)
    return e, t
