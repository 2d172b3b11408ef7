"""numpy restatement of the lockstep fast path's (bitseq / Ising, TB) bf16 numerics, driven by
the device's OWN forward (activation images, ReLU masks, log-softmax record) — TEST HELPER.

With the forward fixed to the device's, ReLU units whose pre-activation sits within fp32
rounding of zero cannot flip between the device and the model, so the backward (dlogits,
dgrad chain, weight and bias gradients) is compared at fp32-summation accuracy. The forward
itself is compared separately, element by element, against the bf16 operand model.

Rounding points (lockstep.cu): logits bf16(h W + b); dlogits g (onehot - exp(x - lse)) over
legal columns, fp32 then bf16 for the GEMM operands, the head-bias sum over the fp32 values;
dz_l = bf16(mask_l (dz_{l+1} W_{l+1}^T)) with the bias sums over the fp32 masked values; the
one-hot layer-1 operand of dW1 in bf16 (the bitseq filled-count feature is fractional).
"""
from __future__ import annotations

import numpy as np

H = 256


def bf16(x):
    """Round-to-nearest-even to bf16 of the fp32 value (cvt.rn.bf16.f32)."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def decode_image(buf: np.ndarray, rows: int, cols: int, kblocks: int | None = None) -> np.ndarray:
    """[rows x cols] from 128-row tile images, 64-column blocks, 128B swizzle (sw128_offset)."""
    u16 = buf.view(np.uint16)
    kb = kblocks if kblocks is not None else cols // 64
    r = np.arange(rows)[:, None]
    c = np.arange(cols)[None, :]
    m, row = r // 128, r % 128
    blk, cc = c >> 6, c & 63
    chunk = (cc >> 3) ^ (row & 7)
    off = (m * kb + blk) * (128 * 128) + row * 128 + chunk * 16 + (cc & 7) * 2
    return (u16[off // 2].astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def unpack_mask(buf: np.ndarray, rows: int) -> np.ndarray:
    return np.unpackbits(buf.reshape(rows, H // 8), axis=1, bitorder="little").astype(bool)


def split_params(p, obs_dim, n_hidden, A):
    off, W, b = 0, [], []
    dims = [obs_dim] + [H] * n_hidden
    for l in range(n_hidden):
        W.append(p[off:off + dims[l] * H].reshape(dims[l], H))
        off += dims[l] * H
        b.append(p[off:off + H])
        off += H
    Wf = p[off:off + H * A].reshape(H, A)
    off += H * A
    return W, b, Wf, p[off:off + A], off + A


def rows_obs_mask(oracle, actions):
    """Observation and legal-action mask of every row r = t * B + b (step-major)."""
    B, T = actions.shape
    sh = oracle.shape
    obs = np.zeros((B * T, sh.obs_dim))
    mask = np.zeros((B * T, sh.num_actions), bool)
    for t in range(T):
        for b in range(B):
            o, m = oracle.obs_after(actions[b, :t])
            obs[t * B + b] = o
            mask[t * B + b] = m > 0
    return obs, mask


def backward_given_forward(p, n_params, obs, mask, actions, bufs, n_hidden):
    """Flat gradient of the device's TB backward from the device's forward record."""
    B, T = actions.shape
    R, A = mask.shape
    W, bias, Wf, bfw, off_end = split_params(p, obs.shape[1], n_hidden, A)
    hs = [decode_image(bufs[f"h{l}"], R, H) for l in range(n_hidden)]
    masks = [unpack_mask(bufs[f"mask{l}"], R) for l in range(n_hidden)]
    rec = bufs["rowbuf"].view(np.float32).reshape(R, 2).astype(np.float64)
    coef = bufs["coef"].view(np.float32).astype(np.float64)
    act = actions.T.reshape(-1)  # row r = t * B + b
    x = bf16(hs[-1] @ bf16(Wf) + bfw)
    dlog = np.where(mask, -coef[:, None] * np.exp(x - rec[:, 1:2]), 0.0)
    dlog[np.arange(R), act] += coef
    dlog_q = bf16(dlog)
    g = np.zeros(n_params)
    off = 0
    offs = []
    for l in range(n_hidden):
        offs.append(off)
        off += W[l].size + H
    g[off:off + Wf.size] = (hs[-1].T @ dlog_q).reshape(-1)
    g[off + Wf.size:off + Wf.size + A] = dlog.sum(0)
    dh = dlog_q @ bf16(Wf).T
    for l in range(n_hidden - 1, -1, -1):
        dz = np.where(masks[l], dh, 0.0)
        dz_q = bf16(dz)
        hin = hs[l - 1] if l > 0 else bf16(obs)
        g[offs[l]:offs[l] + W[l].size] = (hin.T @ dz_q).reshape(-1)
        g[offs[l] + W[l].size:offs[l] + W[l].size + H] = dz.sum(0)
        if l > 0:
            dh = dz_q @ bf16(W[l]).T
    return g, hs, masks


def forward_model(p, obs, n_hidden, A, ising_l1: bool):
    """The bf16 operand model's activations (fp64 arithmetic on bf16 operands)."""
    W, bias, Wf, bfw, _ = split_params(p, obs.shape[1], n_hidden, A)
    hs, x = [], obs
    for l in range(n_hidden):
        if l == 0 and ising_l1:  # persistent Ising layer 1 (k_ls_ising_l1img / k_ls_h1init)
            W1 = W[0]
            z = np.tile(bias[0] + bf16(W1[2::3]).sum(0), (obs.shape[0], 1))
            for s in range(obs.shape[1] // 3):
                for u in (0, 1):
                    sel = obs[:, 3 * s + u] > 0
                    z[sel] += bf16(bf16(W1[3 * s + u]) - bf16(W1[3 * s + 2]))
        else:
            z = x @ bf16(W[l]) + bias[l]
        x = bf16(np.maximum(z, 0.0))
        hs.append(x)
    return hs
