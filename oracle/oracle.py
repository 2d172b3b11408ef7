"""ctypes front-ends for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``   — the plain-C restatement (oracle/liboracle.so, gfn_oracle.c).
* ``RefLib``   — the unmodified reference library + shim (oracle/_ref/libgfnref*.so).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs
import this module. The product (paper_2511_16592_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2511_16592_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; _ref only when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        P = C.POINTER
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [P(abi.EnvDesc), P(abi.TrainDesc), C.c_int32, C.c_int32,
                                 C.c_char_p, C.c_int32]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.c_void_p]
        L.orc_shape.argtypes = [C.c_void_p, P(abi.EnvShape)]
        L.orc_num_params.restype = C.c_int64
        L.orc_num_params.argtypes = [C.c_void_p]
        for f in ("orc_get_params", "orc_get_grads"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_set_params.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        L.orc_set_grads.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        L.orc_get_adam.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.orc_set_adam.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_double,
                                   C.c_double, C.c_int64]
        L.orc_rollout.argtypes = [C.c_void_p, C.c_int64, C.c_double]
        L.orc_replay.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_rollout_uniform.argtypes = [C.c_void_p, C.c_int64]
        L.orc_model_grads.argtypes = [C.c_void_p, C.c_double, C.c_int32] + [C.c_void_p] * 4
        L.orc_teacher_actions.argtypes = [C.c_void_p, C.c_int64, C.c_double, C.c_void_p]
        L.orc_local_counts.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_compute_grads.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
        L.orc_apply_adam.argtypes = [C.c_void_p, C.c_double]
        L.orc_iteration.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_mlp_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_obs_after.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]
        L.orc_log_reward_of_state.restype = C.c_double
        L.orc_log_reward_of_state.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_bitseq_modes.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.orc_dag_cache.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.orc_dag_true_adj.argtypes = [C.c_void_p, C.c_void_p]
        L.orc_threefry2x64.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_fold_in.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
        L.orc_uniform_scalar.restype = C.c_double
        L.orc_uniform_scalar.argtypes = [C.c_void_p]
        L.orc_categorical.restype = C.c_int32
        L.orc_categorical.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.orc_eps_uniform.restype = C.c_int32
        L.orc_eps_uniform.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_void_p]
        L.orc_schedule_value.restype = C.c_double
        L.orc_schedule_value.argtypes = [P(abi.Schedule), C.c_int64]
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


# ---------------- RNG helpers ----------------
def threefry(key, c0, c1):
    k = np.array(key, dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lib().orc_threefry2x64(_p(k), c0, c1, _p(out))
    return int(out[0]), int(out[1])


def fold_in(key, idx):
    k = np.array(key, dtype=np.uint64)
    out = np.zeros(2, dtype=np.uint64)
    lib().orc_fold_in(_p(k), idx, _p(out))
    return int(out[0]), int(out[1])


def uniform_scalar(key):
    k = np.array(key, dtype=np.uint64)
    return lib().orc_uniform_scalar(_p(k))


# bf16 operand model flags (gfn_oracle.h ORC_BFM_*)
BFM_W, BFM_ACT, BFM_GRAD, BFM_LOGIT, BFM_ISING_L1 = 1, 2, 4, 8, 16
BFM_FUSED = BFM_W | BFM_ACT | BFM_GRAD             # hypergrid / DAG fast path
BFM_LOCKSTEP = BFM_FUSED | BFM_LOGIT                # bitseq, Ising per-step path


def param_tensors(oracle) -> list:
    """(name, begin, end) of every tensor of the flat parameter vector in MlpParams::tensors()
    order (nn.cpp:8-19): trunk W1, b1, ..., fwd head, bwd head, flow head."""
    sh, t = oracle.shape, oracle.train
    dims = [sh.obs_dim] + [t.hidden[i] for i in range(t.num_hidden)]
    sizes = []
    for i in range(t.num_hidden):
        sizes += [(f"W{i + 1}", dims[i] * dims[i + 1]), (f"b{i + 1}", dims[i + 1])]
    H = dims[-1]
    for nm, k in (("fwd", sh.num_actions), ("bwd", sh.num_backward_actions), ("flow", 1)):
        sizes += [(f"W{nm}", H * k), (f"b{nm}", k)]
    out, off = [], 0
    for nm, k in sizes:
        out.append((nm, off, off + k))
        off += k
    assert off == oracle.n_params
    return out


def make_key(seed):
    return (0x9E3779B97F4A7C15, seed)


class Oracle:
    """The restatement, one rank slice [b0, b0+nb) of the global batch."""

    def __init__(self, env: abi.EnvDesc, train: abi.TrainDesc, b0: int = 0, nb: int = 0):
        err = C.create_string_buffer(256)
        self.env, self.train = env, train
        self.h = lib().orc_create(C.byref(env), C.byref(train), b0, nb, err, 256)
        if not self.h:
            raise ValueError(err.value.decode())
        sh = abi.EnvShape()
        lib().orc_shape(self.h, C.byref(sh))
        self.shape = sh
        self.n_params = lib().orc_num_params(self.h)
        self.nb = nb if nb > 0 else train.batch_size

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(lib().orc_last_error(self.h).decode())

    def params(self):
        p = np.zeros(self.n_params)
        z = C.c_double()
        lib().orc_get_params(self.h, _p(p), C.byref(z))
        return p, z.value

    def set_params(self, p, log_z):
        p = np.ascontiguousarray(p, dtype=np.float64)
        lib().orc_set_params(self.h, _p(p), log_z)

    def adam(self):
        m = np.zeros(self.n_params)
        v = np.zeros(self.n_params)
        t, zt = C.c_int64(), C.c_int64()
        zm, zv = C.c_double(), C.c_double()
        lib().orc_get_adam(self.h, _p(m), _p(v), C.byref(t), C.byref(zm), C.byref(zv), C.byref(zt))
        return m, v, t.value, zm.value, zv.value, zt.value

    def set_adam(self, m, v, t, zm, zv, zt):
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        lib().orc_set_adam(self.h, _p(m), _p(v), t, zm, zv, zt)

    def rollout(self, it, eps):
        self._check(lib().orc_rollout(self.h, it, eps))

    def rollout_uniform(self, it):
        """eps = 1 rollout without the policy forward (identical draws, see gfn_oracle.c)."""
        self._check(lib().orc_rollout_uniform(self.h, it))

    def model_grads(self, flags, norm=0.0):
        """bf16 operand model (BFM_* flags): (loss, grads, dlogz, row log pi_F [nb, T])."""
        loss, dz = C.c_double(), C.c_double()
        g = np.zeros(self.n_params)
        lp = np.zeros((self.nb, self.shape.max_traj_len))
        self._check(lib().orc_model_grads(self.h, norm, flags, C.byref(loss), _p(g), C.byref(dz), _p(lp)))
        return loss.value, g, dz.value, lp

    def teacher_actions(self, it, eps):
        """Actions of the fp64 reference sampler at every state of the resident batch."""
        out = np.zeros((self.nb, self.shape.max_traj_len), dtype=np.int32)
        self._check(lib().orc_teacher_actions(self.h, it, eps, _p(out)))
        return out

    def replay(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.int32)
        self._check(lib().orc_replay(self.h, _p(a)))

    def counts(self):
        s, m = C.c_int64(), C.c_int64()
        lib().orc_local_counts(self.h, C.byref(s), C.byref(m))
        return s.value, m.value

    def compute_grads(self, norm=0.0):
        loss = C.c_double()
        self._check(lib().orc_compute_grads(self.h, norm, C.byref(loss)))
        return loss.value

    def grads(self):
        g = np.zeros(self.n_params)
        dz = C.c_double()
        lib().orc_get_grads(self.h, _p(g), C.byref(dz))
        return g, dz.value

    def set_grads(self, g, dz):
        g = np.ascontiguousarray(g, dtype=np.float64)
        lib().orc_set_grads(self.h, _p(g), dz)

    def apply_adam(self, lr):
        lib().orc_apply_adam(self.h, lr)

    def iteration(self, it):
        loss = C.c_double()
        self._check(lib().orc_iteration(self.h, it, C.byref(loss)))
        return loss.value

    def schedule(self, which, it):
        s = getattr(self.train, which)
        return lib().orc_schedule_value(C.byref(s), it)

    def batch(self):
        nb, T, sw = self.nb, self.shape.max_traj_len, self.shape.state_words

        class View(C.Structure):
            _fields_ = [("nb", C.c_int32), ("T", C.c_int32), ("sw", C.c_int32),
                        ("lengths", C.c_void_p), ("fwd", C.c_void_p), ("bwd", C.c_void_p),
                        ("logr", C.c_void_p), ("logpb", C.c_void_p), ("delta", C.c_void_p),
                        ("term", C.c_void_p)]
        v = View()
        lib().orc_batch.argtypes = [C.c_void_p, C.c_void_p]
        lib().orc_batch(self.h, C.byref(v))

        def arr(ptr, n, ct, dt):
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).astype(dt).copy()
        return dict(
            lengths=arr(v.lengths, nb, C.c_int32, np.int32),
            fwd_actions=arr(v.fwd, nb * T, C.c_int32, np.int32).reshape(nb, T),
            bwd_actions=arr(v.bwd, nb * T, C.c_int32, np.int32).reshape(nb, T),
            log_rewards=arr(v.logr, nb, C.c_double, np.float64),
            log_pb=arr(v.logpb, nb * T, C.c_double, np.float64).reshape(nb, T),
            delta=arr(v.delta, nb * T, C.c_double, np.float64).reshape(nb, T),
            terminal_state=arr(v.term, nb * sw, C.c_uint32, np.uint32).reshape(nb, sw),
        )

    def mlp_forward(self, obs):
        obs = np.ascontiguousarray(obs, dtype=np.float64)
        n = obs.shape[0]
        lg = np.zeros((n, self.shape.num_actions))
        fl = np.zeros(n)
        lib().orc_mlp_forward(self.h, _p(obs), n, _p(lg), _p(fl))
        return lg, fl

    def obs_after(self, actions):
        a = np.ascontiguousarray(actions, dtype=np.int32)
        obs = np.zeros(self.shape.obs_dim)
        mask = np.zeros(self.shape.num_actions, dtype=np.uint8)
        lib().orc_obs_after(self.h, _p(a), len(a), _p(obs), _p(mask))
        return obs, mask

    def log_reward_of_state(self, packed):
        w = np.ascontiguousarray(packed, dtype=np.uint32)
        return lib().orc_log_reward_of_state(self.h, _p(w))

    def bitseq_modes(self):
        n = self.env.bs_n_bits
        buf = np.zeros((4096, n), dtype=np.uint8)
        cnt = lib().orc_bitseq_modes(self.h, _p(buf), 4096)
        return buf[:cnt].copy()

    def dag_cache(self):
        d = self.env.dag_d
        out = np.zeros(d << d)
        lib().orc_dag_cache(self.h, _p(out), d << d)
        return out.reshape(d, 1 << d)

    def dag_true_adj(self):
        out = np.zeros(16, dtype=np.uint32)
        n = lib().orc_dag_true_adj(self.h, _p(out))
        return out[:n].copy()


# ---------------- the compiled reference (oracle/_ref) ----------------
_REF = {}


def ref_available(kind: str = "port") -> bool:
    name = "libgfnref.so" if kind == "port" else "libgfnref_fast.so"
    return os.path.exists(os.path.join(HERE, "_ref", name))


def ref_lib(kind: str = "port"):
    if kind not in _REF:
        name = "libgfnref.so" if kind == "port" else "libgfnref_fast.so"
        L = C.CDLL(os.path.join(HERE, "_ref", name))
        P = C.POINTER
        L.ref_create.restype = C.c_void_p
        L.ref_create.argtypes = [P(abi.EnvDesc), P(abi.TrainDesc)]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [C.c_void_p]
        L.ref_rollout.argtypes = [C.c_void_p, C.c_int64, C.c_double]
        L.ref_batch.argtypes = [C.c_void_p] + [C.c_void_p] * 6
        L.ref_terminal_keys.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_compute_grads.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_num_params.restype = C.c_int64
        L.ref_num_params.argtypes = [C.c_void_p]
        L.ref_get_grads.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_apply_adam.argtypes = [C.c_void_p, C.c_double]
        L.ref_get_params.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_set_params.argtypes = [C.c_void_p, C.c_void_p, C.c_double]
        L.ref_iteration.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.ref_uniform_fold.restype = C.c_double
        L.ref_uniform_fold.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_threefry.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p]
        L.ref_run_bench.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_int,
                                    C.c_void_p, C.c_void_p]
        L.ref_exact_divergence.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_pearson.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_void_p]
        L.ref_mc_logprob.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p]
        L.ref_backward_rollout.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64]
        L.ref_save_checkpoint.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_load_checkpoint.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
        _REF[kind] = L
    return _REF[kind]


class RefLib:
    """The unmodified reference through its public API (oracle/ref_shim.cpp)."""

    def __init__(self, env: abi.EnvDesc, train: abi.TrainDesc, kind: str = "port"):
        self.L = ref_lib(kind)
        self.env, self.train = env, train
        self.h = self.L.ref_create(C.byref(env), C.byref(train))
        if not self.h:
            raise ValueError(self.L.ref_last_error(None).decode())
        self.n_params = self.L.ref_num_params(self.h)
        self.B = train.batch_size

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_destroy(self.h)
            self.h = None

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.L.ref_last_error(self.h).decode())

    def rollout(self, it, eps):
        self._check(self.L.ref_rollout(self.h, it, eps))

    def batch(self, T):
        B = self.B
        out = dict(lengths=np.zeros(B, np.int32), fwd_actions=np.zeros((B, T), np.int32),
                   bwd_actions=np.zeros((B, T), np.int32), log_rewards=np.zeros(B),
                   log_pb=np.zeros((B, T)), delta=np.zeros((B, T)))
        self.L.ref_batch(self.h, *[_p(out[k]) for k in ("lengths", "fwd_actions", "bwd_actions",
                                                        "log_rewards", "log_pb", "delta")])
        buf = C.create_string_buffer(1 << 24)
        n = self.L.ref_terminal_keys(self.h, buf, 1 << 24)
        out["terminal_keys"] = buf.value[:n].decode().split("\n")[:-1]
        return out

    def compute_grads(self):
        loss = C.c_double()
        self._check(self.L.ref_compute_grads(self.h, C.byref(loss)))
        return loss.value

    def grads(self):
        g = np.zeros(self.n_params)
        dz = C.c_double()
        self.L.ref_get_grads(self.h, _p(g), C.byref(dz))
        return g, dz.value

    def apply_adam(self, lr):
        self.L.ref_apply_adam(self.h, lr)

    def params(self):
        p = np.zeros(self.n_params)
        z = C.c_double()
        self.L.ref_get_params(self.h, _p(p), C.byref(z))
        return p, z.value

    def set_params(self, p, log_z):
        p = np.ascontiguousarray(p, dtype=np.float64)
        self.L.ref_set_params(self.h, _p(p), log_z)

    def iteration(self, it):
        loss = C.c_double()
        self._check(self.L.ref_iteration(self.h, it, C.byref(loss)))
        return loss.value

    def save_checkpoint(self, path, step):
        self._check(self.L.ref_save_checkpoint(self.h, str(path).encode(), step))

    def load_checkpoint(self, path):
        st = C.c_int64()
        self._check(self.L.ref_load_checkpoint(self.h, str(path).encode(), C.byref(st)))
        return st.value

    def backward_rollout(self, terminal_words, key):
        """backward_rollout (env_core.hpp:314-370) of packed terminals [B, state_words] under
        key = (hi, lo): becomes the session batch (batch() / compute_grads() act on it)."""
        w = np.ascontiguousarray(terminal_words, dtype=np.uint32)
        assert len(w) == self.B
        self._check(self.L.ref_backward_rollout(self.h, w.ctypes.data_as(C.c_void_p), len(w),
                                                int(key[0]), int(key[1])))

    def mc_logprob(self, terminal_words, key, num_samples: int = 10):
        """mc_terminal_logprob (exact.hpp:229-241) of one packed terminal state,
        key = (hi, lo) RngKey words."""
        w = np.ascontiguousarray(terminal_words, dtype=np.uint32)
        d = C.c_double()
        self._check(self.L.ref_mc_logprob(self.h, w.ctypes.data_as(C.c_void_p), num_samples,
                                          int(key[0]), int(key[1]), C.byref(d)))
        return d.value

    def pearson(self, step: int, mc: int = 10, test_seed: int = 1):
        """The bitseq `pearson` metric of the current policy (train.cpp:440-454)."""
        d = C.c_double()
        self._check(self.L.ref_pearson(self.h, step, mc, test_seed, C.byref(d)))
        return d.value

    def exact_divergence(self):
        """TV (hypergrid) / JSD (DAG) of the current policy's exact terminal marginal to the
        target distribution, by the reference's exact enumeration (exact.hpp:76)."""
        d = C.c_double()
        self._check(self.L.ref_exact_divergence(self.h, C.byref(d)))
        return d.value


def ref_eb_gfn(kv: dict, out_dir: str):
    """The reference's run_eb_gfn (train.cpp:875-1018) via its Config front door, in a separate
    process (oracle/_ref/eb_driver). Returns (result dict, coupling [D, D], metrics rows
    [(step, loss, logZ, nlr, accept_rate)]) read back from its %.17g output files."""
    exe = os.path.join(HERE, "_ref", "eb_driver")
    r = subprocess.run([exe, out_dir] + [f"{k}={v}" for k, v in kv.items()], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    init, best, final, loss = (float(x) for x in r.stdout.split())
    with open(os.path.join(out_dir, "coupling.txt")) as f:
        lines = f.read().strip().split("\n")[1:]
    J = np.array([[float(v) for v in ln.split()] for ln in lines])
    rows = []
    with open(os.path.join(out_dir, "metrics.csv")) as f:
        for ln in f.read().strip().split("\n")[1:]:
            rows.append(tuple(float(v) for v in ln.split(",")))
    return dict(init_nlr=init, best_nlr=best, final_nlr=final, final_loss=loss), J, rows


def ref_gibbs_data(side: int, sigma: float, seed: int, n: int, burn_in: int = 2000, thinning: int = 10,
                   chains: int = 1, hottest_beta: float = 0.2, kind: str = "port"):
    """gibbs_data_sampler (ising.cpp:185-220) with key fold_in(make_key(seed), 0x919B)."""
    L = ref_lib(kind)
    L.ref_gibbs_data.argtypes = [C.c_int, C.c_double, C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                 C.c_double, C.c_void_p]
    out = np.zeros((n, side * side), dtype=np.int8)
    rc = L.ref_gibbs_data(side, sigma, seed, n, burn_in, thinning, chains, hottest_beta, _p(out))
    if rc != 0:
        raise RuntimeError(L.ref_last_error(None).decode())
    return out


def ref_run_bench(env_name: str, kv: dict, kind: str = "fast"):
    """The reference's own run_bench (train.cpp:294-334) via its Config front door."""
    L = ref_lib(kind)
    keys = [k.encode() for k in kv]
    vals = [str(v).encode() for v in kv.values()]
    karr = (C.c_char_p * len(keys))(*keys)
    varr = (C.c_char_p * len(vals))(*vals)
    mean, se = C.c_double(), C.c_double()
    rc = L.ref_run_bench(env_name.encode(), C.cast(karr, C.c_void_p), C.cast(varr, C.c_void_p),
                         len(keys), C.byref(mean), C.byref(se))
    if rc != 0:
        raise RuntimeError(L.ref_last_error(None).decode())
    return mean.value, se.value
