"""Host-side mirror of the reference training API over the libgfnx C ABI.

``Trainer`` follows the reference drivers (proj/src/train.cpp): ``forward_rollout``
(env_core.hpp:232-274), ``train_step`` (train.cpp:164-192) and ``iteration``
(the train_scenario loop body, train.cpp:224-229), with the same error classes as
proj/include/gfn/errors.hpp. Everything numeric runs in libgfnx.so on the GPU; there
is no CPU fallback — a missing or unloadable library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgfnx.so")
_LIB = None


class config_error(RuntimeError):
    pass


class contract_violation(RuntimeError):
    pass


class numeric_error(RuntimeError):
    pass


class device_error(RuntimeError):
    pass


_ERRORS = {abi.ERR_CONFIG: config_error, abi.ERR_CONTRACT: contract_violation,
           abi.ERR_NUMERIC: numeric_error, abi.ERR_CUDA: device_error, abi.ERR_NCCL: device_error}


def lib():
    """Load libgfnx.so (built in-tree by __graft_entry__.build / build.py). Fails loudly."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libgfnx.so not built at {LIB_PATH}: run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        vp = C.c_void_p
        L.gfnx_last_error.restype = C.c_char_p
        L.gfnx_last_error.argtypes = [vp]
        L.gfnx_create.argtypes = [P(abi.EnvDesc), P(abi.TrainDesc), C.c_int32, C.c_int32,
                                  C.c_int32, vp, P(vp)]
        L.gfnx_destroy.argtypes = [vp]
        L.gfnx_group_create.argtypes = [C.c_int32, P(vp)]
        L.gfnx_group_destroy.argtypes = [vp]
        L.gfnx_create_in_group.argtypes = [P(abi.EnvDesc), P(abi.TrainDesc), C.c_int32, C.c_int32, vp, P(vp)]
        L.gfnx_nccl_unique_id.argtypes = [vp]
        L.gfnx_env_shape_of.argtypes = [P(abi.EnvDesc), P(abi.EnvShape)]
        L.gfnx_default_env_desc.argtypes = [C.c_int32, P(abi.EnvDesc)]
        L.gfnx_default_train_desc.argtypes = [C.c_int32, P(abi.TrainDesc)]
        L.gfnx_num_params.argtypes = [vp, P(C.c_int64)]
        L.gfnx_set_params.argtypes = [vp, vp, C.c_int64, C.c_double]
        L.gfnx_get_params.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_set_adam_state.argtypes = [vp, vp, vp, C.c_int64, C.c_double, C.c_double, C.c_int64]
        L.gfnx_get_adam_state.argtypes = [vp] + [vp] * 6
        L.gfnx_rollout.argtypes = [vp, C.c_int64, C.c_double]
        L.gfnx_train_step.argtypes = [vp, C.c_double, vp]
        L.gfnx_compute_grads.argtypes = [vp, vp]
        L.gfnx_get_grads.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_export_row_logpf.argtypes = [vp, vp, C.c_int64]
        L.gfnx_log_rewards.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_log_rewards_device.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_debug_buffer.argtypes = [vp, C.c_char_p, vp, C.c_int64, P(C.c_int64)]
        L.gfnx_iteration.argtypes = [vp, C.c_int64, vp]
        L.gfnx_run.argtypes = [vp, C.c_int64, C.c_int64, vp]
        L.gfnx_synchronize.argtypes = [vp]
        L.gfnx_batch_dims.argtypes = [vp, vp, vp, vp, vp]
        L.gfnx_export_batch.argtypes = [vp, P(abi.HostBatch)]
        L.gfnx_kernel_launches.restype = C.c_int64
        L.gfnx_kernel_launches.argtypes = [vp]
        L.gfnx_last_phase_ms.argtypes = [vp, vp, vp]
        L.gfnx_test_threefry.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_test_uniform_fold.argtypes = [C.c_uint64, C.c_uint64, vp, C.c_int64, vp]
        L.gfnx_abi_version.restype = C.c_int32
        L.gfnx_event_record.argtypes = [vp, C.c_int32]
        L.gfnx_event_elapsed.argtypes = [vp, C.c_int32, C.c_int32, vp]
        L.gfnx_profile.argtypes = [vp, C.c_int32]
        L.gfnx_profile_read.restype = C.c_int32
        L.gfnx_profile_read.argtypes = [vp, vp, C.c_int32, vp, vp, C.c_int32]
        L.gfnx_counters.argtypes = [vp, vp, C.c_int32]
        L.gfnx_phase_timers.argtypes = [vp, C.c_int32, vp, C.c_int32]
        L.gfnx_test_mma_rate.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp]
        L.gfnx_test_ts_mma.argtypes = [vp, vp, vp]
        L.gfnx_save_checkpoint.argtypes = [vp, C.c_char_p, C.c_int64]
        L.gfnx_exact_terminal_marginal.argtypes = [vp, vp, C.c_int64, vp]
        L.gfnx_buffer_reset.argtypes = [vp, C.c_int64]
        L.gfnx_mc_terminal_logprob.argtypes = [vp, vp, C.c_int64, C.c_int32, vp, vp]
        L.gfnx_backward_rollout.argtypes = [vp, vp, C.c_int64, C.c_uint64, C.c_uint64]
        L.gfnx_rollout_from_actions.argtypes = [vp, vp, C.c_int64]
        L.gfnx_pearson.argtypes = [vp, C.c_int64, C.c_int32, C.c_uint64, vp]
        L.gfnx_eb_default_desc.argtypes = [P(abi.EbDesc)]
        L.gfnx_eb_init.argtypes = [vp, P(abi.EbDesc), vp, C.c_int64]
        L.gfnx_eb_run.argtypes = [vp, C.c_int64, C.c_int64, vp]
        L.gfnx_eb_coupling.argtypes = [vp, vp, vp, C.c_int64, vp]
        L.gfnx_eb_dataset.argtypes = [vp, vp, C.c_int64]
        L.gfnx_ising_gibbs_data.argtypes = [C.c_int32, C.c_double, C.c_uint64, P(abi.EbDesc), vp, C.c_int64]
        L.gfnx_buffer_push.argtypes = [vp]
        L.gfnx_tv_buffer.argtypes = [vp, vp, vp]
        L.gfnx_load_checkpoint.argtypes = [vp, C.c_char_p, vp]
        L.gfnx_iteration_async.argtypes = [vp, C.c_int64, C.c_int32]
        L.gfnx_slot_wait.argtypes = [vp, C.c_int32, P(abi.SlotView)]
        _LIB = L
    return _LIB


def eb_desc(**kw):
    """run_eb_gfn's defaults (train.cpp:899-913) as a gfnx_eb_desc, with overrides."""
    d = abi.EbDesc()
    lib().gfnx_eb_default_desc(C.byref(d))
    for k, v in kw.items():
        if not hasattr(d, k):
            raise KeyError(k)
        setattr(d, k, v)
    return d


def ising_gibbs_data(side: int, sigma: float, seed: int, n: int, desc=None):
    """gibbs_data_sampler (ising.cpp:185-220) on the true toroidal coupling: [n, side^2] spins."""
    d = desc if desc is not None else eb_desc()
    out = np.zeros((n, side * side), dtype=np.int8)
    _raise(lib().gfnx_ising_gibbs_data(side, sigma, seed, C.byref(d), _p(out), n))
    return out


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _raise(rc, h=None):
    if rc != abi.OK:
        msg = lib().gfnx_last_error(h).decode()
        raise _ERRORS.get(rc, device_error)(msg)


def env_shape(env: abi.EnvDesc) -> abi.EnvShape:
    s = abi.EnvShape()
    _raise(lib().gfnx_env_shape_of(C.byref(env), C.byref(s)))
    return s


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _raise(lib().gfnx_nccl_unique_id(buf))
    return buf.raw


class Group:
    """In-process communicator (gfnx_group): `world` ranks driven by the threads of this
    process; their all-reduce is libgfnx's peer-memory sum kernel instead of NCCL."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _raise(lib().gfnx_group_create(world, C.byref(h)))
        self.h, self.world = h, world

    def close(self):
        if getattr(self, "h", None):
            _raise(lib().gfnx_group_destroy(self.h))
            self.h = None


class Trainer:
    """One rank's device engine (one gfnx_ctx)."""

    def __init__(self, env: abi.EnvDesc, train: abi.TrainDesc, device: int = 0, rank: int = 0,
                 world: int = 1, nccl_id: bytes | None = None, group: Group | None = None):
        self.env, self.train = env, train
        h = C.c_void_p()
        if group is not None:
            _raise(lib().gfnx_create_in_group(C.byref(env), C.byref(train), device, rank, group.h,
                                              C.byref(h)))
        else:
            idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
            _raise(lib().gfnx_create(C.byref(env), C.byref(train), device, rank, world, idbuf,
                                     C.byref(h)))
        self.h = h
        n = C.c_int64()
        lib().gfnx_num_params(h, C.byref(n))
        self.n_params = n.value
        self.shape = env_shape(env)
        bl, b0, T, sw = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        lib().gfnx_batch_dims(h, C.byref(bl), C.byref(b0), C.byref(T), C.byref(sw))
        self.local_batch, self.first_traj, self.T, self.state_words = bl.value, b0.value, T.value, sw.value

    def close(self):
        if getattr(self, "h", None):
            lib().gfnx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        _raise(rc, self.h)

    # -- parameters / optimizer state (MlpParams::tensors() order, nn.cpp:8-19) --
    def params(self):
        p = np.zeros(self.n_params)
        z = C.c_double()
        self._check(lib().gfnx_get_params(self.h, _p(p), self.n_params, C.byref(z)))
        return p, z.value

    def set_params(self, p, log_z):
        p = np.ascontiguousarray(p, dtype=np.float64)
        self._check(lib().gfnx_set_params(self.h, _p(p), self.n_params, log_z))

    def adam_state(self):
        m, v = np.zeros(self.n_params), np.zeros(self.n_params)
        t, zt = C.c_int64(), C.c_int64()
        zm, zv = C.c_double(), C.c_double()
        self._check(lib().gfnx_get_adam_state(self.h, _p(m), _p(v), C.byref(t), C.byref(zm),
                                              C.byref(zv), C.byref(zt)))
        return m, v, t.value, zm.value, zv.value, zt.value

    def set_adam_state(self, m, v, t, zm, zv, zt):
        m = np.ascontiguousarray(m, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        self._check(lib().gfnx_set_adam_state(self.h, _p(m), _p(v), t, zm, zv, zt))

    # -- GFNCKPT1 checkpoints (checkpoint.cpp:11-107) --
    def save_checkpoint(self, path, step: int = 0):
        self._check(lib().gfnx_save_checkpoint(self.h, str(path).encode(), step))

    def load_checkpoint(self, path) -> int:
        st = C.c_int64()
        self._check(lib().gfnx_load_checkpoint(self.h, str(path).encode(), C.byref(st)))
        return st.value

    def exact_terminal_marginal(self, n_cells: int):
        """(marginal over cells, TV to R/Z) of the current policy (hypergrid, device DP)."""
        m = np.zeros(n_cells)
        tv = C.c_double()
        self._check(lib().gfnx_exact_terminal_marginal(self.h, _p(m), n_cells, C.byref(tv)))
        return m, tv.value

    def mc_terminal_logprob(self, terminals, keys, num_samples: int = 10):
        """mc_terminal_logprob (exact.hpp:229-241) of packed terminal states [n, state_words];
        keys [n, 2] uint64 RngKey words (one backward-rollout key per terminal)."""
        t = np.ascontiguousarray(terminals, dtype=np.uint32)
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        out = np.zeros(len(t))
        self._check(lib().gfnx_mc_terminal_logprob(self.h, _p(t), len(t), num_samples, _p(k), _p(out)))
        return out

    def buffer_reset(self, capacity: int = 200000):
        """New empty terminal-state FIFO (FifoBuffer, buffer.hpp:13-55) for `tv_buffer`."""
        self._check(lib().gfnx_buffer_reset(self.h, capacity))

    def buffer_push(self):
        """buffer.push_batch(batch.terminal_keys) of the resident batch (train.cpp:231)."""
        self._check(lib().gfnx_buffer_push(self.h))

    def tv_buffer(self):
        """(buffer size, tv_distance(buffer.empirical(), exact)) (metrics.cpp:35-48)."""
        n, tv = C.c_int64(), C.c_double()
        self._check(lib().gfnx_tv_buffer(self.h, C.byref(n), C.byref(tv)))
        return n.value, tv.value

    # -- the hot path --
    def forward_rollout(self, it: int, eps: float):
        self._check(lib().gfnx_rollout(self.h, it, eps))

    def backward_rollout(self, terminals, key):
        """backward_rollout (env_core.hpp:314-370) of local_batch packed terminal states
        [n, state_words] under key = (hi, lo): the resident batch (forward orientation)."""
        t = np.ascontiguousarray(terminals, dtype=np.uint32)
        self._check(lib().gfnx_backward_rollout(self.h, _p(t), len(t), int(key[0]), int(key[1])))

    def pearson(self, step: int, mc: int = 10, test_seed: int = 1) -> float:
        """The bitseq `pearson` metric (train.cpp:440-454), entirely on the device."""
        d = C.c_double()
        self._check(lib().gfnx_pearson(self.h, step, mc, test_seed, C.byref(d)))
        return d.value

    # -- EB-GFN (run_eb_gfn, train.cpp:875-1018) --
    def eb_init(self, desc=None, data=None):
        """Start an EB-GFN run (Ising ctx); data: None (Gibbs sampler) or [n, D] spins."""
        d = desc if desc is not None else eb_desc()
        if data is None:
            self._check(lib().gfnx_eb_init(self.h, C.byref(d), None, 0))
        else:
            a = np.ascontiguousarray(data, dtype=np.int8)
            self._check(lib().gfnx_eb_init(self.h, C.byref(d), _p(a), len(a)))

    def eb_run(self, it0: int, n: int):
        """Iterations it0..it0+n-1; returns [n, 4] rows (loss, logZ, neg_log_rmse, accepted)."""
        out = np.zeros((n, 4))
        self._check(lib().gfnx_eb_run(self.h, it0, n, _p(out)))
        return out

    def eb_coupling(self):
        """(J_model, J_true, initial neg_log_rmse)."""
        D = self.env.is_side * self.env.is_side
        jm, jt, z = np.zeros((D, D)), np.zeros((D, D)), C.c_double()
        self._check(lib().gfnx_eb_coupling(self.h, _p(jm), _p(jt), D * D, C.byref(z)))
        return jm, jt, z.value

    def eb_dataset(self, n: int):
        D = self.env.is_side * self.env.is_side
        out = np.zeros((n, D), dtype=np.int8)
        self._check(lib().gfnx_eb_dataset(self.h, _p(out), out.size))
        return out

    def rollout_from_actions(self, actions):
        """rollout_from_actions (env_core.hpp:166-229): actions [local_batch, T], -1 padded."""
        a = np.ascontiguousarray(actions, dtype=np.int32)
        self._check(lib().gfnx_rollout_from_actions(self.h, _p(a), a.size))

    def train_step(self, lr: float, read_loss: bool = True):
        loss = C.c_double()
        self._check(lib().gfnx_train_step(self.h, lr, C.byref(loss) if read_loss else None))
        return loss.value if read_loss else None

    def compute_grads(self):
        loss = C.c_double()
        self._check(lib().gfnx_compute_grads(self.h, C.byref(loss)))
        return loss.value

    def grads(self):
        g = np.zeros(self.n_params)
        dz = C.c_double()
        self._check(lib().gfnx_get_grads(self.h, _p(g), self.n_params, C.byref(dz)))
        return g, dz.value

    def row_logpf(self):
        """Per-row log pi_F(a_t | s_t) [local_batch, T] of the last training pass."""
        out = np.zeros((self.local_batch, self.T))
        self._check(lib().gfnx_export_row_logpf(self.h, _p(out), out.size))
        return out

    def log_rewards(self, states):
        """log_reward_of for packed terminal states [n, state_words] (host arrays)."""
        st = np.ascontiguousarray(states, dtype=np.uint32)
        out = np.zeros(len(st))
        self._check(lib().gfnx_log_rewards(self.h, _p(st), len(st), _p(out)))
        return out

    def log_rewards_device(self, states_soa_ptr: int, n: int, out_ptr: int):
        """Device pointers: word-major states [state_words][n] -> out[n] (stream-ordered)."""
        self._check(lib().gfnx_log_rewards_device(self.h, C.c_void_p(states_soa_ptr), n, C.c_void_p(out_ptr)))

    def debug_buffer(self, name: str) -> np.ndarray:
        """Raw bytes of an internal device buffer (diagnostics; see gfnx_debug_buffer)."""
        n = C.c_int64()
        self._check(lib().gfnx_debug_buffer(self.h, name.encode(), None, 0, C.byref(n)))
        out = np.zeros(n.value, dtype=np.uint8)
        self._check(lib().gfnx_debug_buffer(self.h, name.encode(), _p(out), n.value, C.byref(n)))
        return out

    def iteration(self, it: int, read_loss: bool = True):
        loss = C.c_double()
        self._check(lib().gfnx_iteration(self.h, it, C.byref(loss) if read_loss else None))
        return loss.value if read_loss else None

    def run(self, it0: int, n: int, read_losses: bool = False):
        losses = np.zeros(n) if read_losses else None
        self._check(lib().gfnx_run(self.h, it0, n, _p(losses) if read_losses else None))
        return losses

    def synchronize(self):
        self._check(lib().gfnx_synchronize(self.h))

    def batch(self, fields=None):
        """Host copy of the resident TrajectoryBatch fields (trajectory.hpp:15-33)."""
        B, T, sw = self.local_batch, self.T, self.state_words
        out = dict(lengths=np.zeros(B, np.int32), fwd_actions=np.zeros((B, T), np.int32),
                   bwd_actions=np.zeros((B, T), np.int32), log_rewards=np.zeros(B),
                   log_pb=np.zeros((B, T)), delta=np.zeros((B, T)),
                   terminal_state=np.zeros((B, sw), np.uint32))
        if fields is not None:
            out = {k: v for k, v in out.items() if k in fields}
        hb = abi.HostBatch()
        ptr = {"lengths": C.c_int32, "fwd_actions": C.c_int32, "bwd_actions": C.c_int32,
               "log_rewards": C.c_double, "log_pb": C.c_double, "delta": C.c_double,
               "terminal_state": C.c_uint32}
        field = {"delta": "delta_log_reward"}
        for k, v in out.items():
            setattr(hb, field.get(k, k), v.ctypes.data_as(C.POINTER(ptr[k])))
        self._check(lib().gfnx_export_batch(self.h, C.byref(hb)))
        return out

    def iteration_async(self, it: int, slot: int):
        """Enqueue iteration `it` + D2H of its results into pinned slot `slot` (no wait)."""
        self._check(lib().gfnx_iteration_async(self.h, it, slot))

    def slot_wait(self, slot: int, copy: bool = True):
        """Wait for a slot; returns (it, loss, {lengths, log_rewards, terminal_state})."""
        v = abi.SlotView()
        self._check(lib().gfnx_slot_wait(self.h, slot, C.byref(v)))
        n, sw = v.n, v.state_words
        arr = {"lengths": np.ctypeslib.as_array(v.lengths, shape=(n,)),
               "log_rewards": np.ctypeslib.as_array(v.log_rewards, shape=(n,)),
               "terminal_state": np.ctypeslib.as_array(v.terminal_state, shape=(n, sw))}
        if copy:
            arr = {k: a.copy() for k, a in arr.items()}
        return v.it, v.loss, arr

    def event_record(self, slot: int):
        self._check(lib().gfnx_event_record(self.h, slot))

    def event_elapsed(self, a: int, b: int) -> float:
        ms = C.c_double()
        self._check(lib().gfnx_event_elapsed(self.h, a, b, C.byref(ms)))
        return ms.value

    def profile(self, mode: int):
        """Per-kernel CUDA-event brackets: 0 off, 1 every kernel, 2 the rollout kernel only."""
        self._check(lib().gfnx_profile(self.h, int(mode)))

    def profile_read(self):
        names = C.create_string_buffer(4096)
        ms = np.zeros(64)
        cnt = np.zeros(64, dtype=np.int32)
        n = lib().gfnx_profile_read(self.h, names, 4096, _p(ms), _p(cnt), 64)
        keys = names.value.decode().split("\n")[:n]
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}

    def counters(self):
        out = np.zeros(4, dtype=np.int64)
        self._check(lib().gfnx_counters(self.h, _p(out), 4))
        return [int(x) for x in out]

    PHASES = ("loop_barrier", "layer1", "hidden_mma", "hidden_epilogue", "head_mma", "sample_step",
              "tile_steps", "active_slot_steps", "sample_step_max", "wgrad_pass_a", "wgrad_pass_b",
              "wgrad_pass_c", "sample_sampler", "sample_envstep", "sample_features", "bwd_wait_dlogits",
              "bwd_head", "bwd_dz2", "bwd_w2mma_db2", "bwd_dz1", "bwd_tiles", "bwd_rowload",
              "persist_hid_wimg", "persist_hid_mma", "persist_hid_epi")

    def phase_timers(self, mode: int):
        """Rollout phase clocks (diagnostic): 1 enable, 0 disable, 2 read + clear -> dict."""
        out = np.zeros(len(self.PHASES), dtype=np.int64)
        self._check(lib().gfnx_phase_timers(self.h, mode, _p(out), len(self.PHASES)))
        return dict(zip(self.PHASES, (int(x) for x in out))) if mode == 2 else None

    def kernel_launches(self) -> int:
        return lib().gfnx_kernel_launches(self.h)

    def last_phase_ms(self):
        a, b = C.c_double(), C.c_double()
        self._check(lib().gfnx_last_phase_ms(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value


def test_threefry(keys: np.ndarray, ctrs: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, dtype=np.uint64)
    ctrs = np.ascontiguousarray(ctrs, dtype=np.uint64)
    out = np.zeros_like(keys)
    _raise(lib().gfnx_test_threefry(_p(keys), _p(ctrs), keys.shape[0], _p(out)))
    return out


def test_uniform_fold(key, idx: np.ndarray) -> np.ndarray:
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.zeros(idx.shape[0])
    _raise(lib().gfnx_test_uniform_fold(key[0], key[1], _p(idx), idx.shape[0], _p(out)))
    return out
