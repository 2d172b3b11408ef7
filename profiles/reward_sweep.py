"""batched terminal-reward kernels, B sweep up to 2^24 terminals.

Word-major packed terminal states generated on the device (torch), scored by
gfnx_log_rewards_device; achieved HBM GB/s = algorithmic bytes (state words read + 8 B written
per terminal) / kernel time (CUDA events on the ctx stream, median of reps). Inputs at the
largest sizes exceed the 126 MB L2; smaller sizes are reported as measured (L2-resident after
the first rep)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_16592_b200 import abi, engine  # noqa: E402

ENVS = {
    "hypergrid_20^4": lambda: abi.config("hypergrid_tb_b16"),
    "bitseq_n120_k8": lambda: (abi.env_desc(abi.BITSEQ, bs_n_bits=120, bs_k=8), abi.train_desc(abi.BITSEQ, batch=128)),
    "ising_10x10": lambda: (abi.env_desc(abi.ISING, is_side=10, is_sigma=0.2), abi.train_desc(abi.ISING, batch=128)),
    "dag_d5_bge": lambda: abi.config("dag_mdb_b8192"),
}


def states(e, n, SW, g):
    """[SW][n] int32 (bit patterns) of random terminal states on the device."""
    s = torch.zeros((SW, n), dtype=torch.int32, device="cuda")
    if e.kind == abi.HYPERGRID:
        c = torch.randint(0, e.hg_side, (e.hg_dim, n), generator=g, device="cuda", dtype=torch.int32)
        for i in range(e.hg_dim):
            s[0] |= c[i] << (8 * i)
    elif e.kind == abi.BITSEQ:
        slots = e.bs_n_bits // e.bs_k
        tw = (slots + 3) // 4
        s[:tw] = torch.randint(-2**31, 2**31 - 1, (tw, n), generator=g, device="cuda", dtype=torch.int32)
        if slots % 4:
            s[tw - 1] &= (1 << (8 * (slots % 4))) - 1
        s[tw] = (1 << slots) - 1
    elif e.kind == abi.ISING:
        D = e.is_side ** 2
        nw = SW // 2
        for k in range(nw):
            bits = min(32, D - 32 * k)
            full = -1 if bits == 32 else (1 << bits) - 1
            s[k] = full
            s[nw + k] = torch.randint(-2**31, 2**31 - 1, (n,), generator=g, device="cuda", dtype=torch.int32) & full
    else:  # DAG: random upper-triangular adjacency (acyclic)
        d = e.dag_d
        for u in range(d):
            row = torch.randint(0, 1 << d, (n,), generator=g, device="cuda", dtype=torch.int32)
            row &= ~((1 << (u + 1)) - 1) & ((1 << d) - 1)
            s[u >> 1] |= row << (16 * (u & 1))
    return s


def sweep(sizes=(1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24), reps=20, device=0, peak_gbs=None):
    out = {}
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    for name, mk in ENVS.items():
        e, t = mk()
        tr = engine.Trainer(e, t, device=device)
        SW = tr.state_words
        rows = []
        for n in sizes:
            st = states(e, n, SW, g)
            res = torch.empty(n, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            tr.log_rewards_device(st.data_ptr(), n, res.data_ptr())  # warm-up
            tr.synchronize()
            times = []
            for _ in range(reps):
                tr.event_record(0)
                tr.log_rewards_device(st.data_ptr(), n, res.data_ptr())
                tr.event_record(1)
                tr.synchronize()
                times.append(tr.event_elapsed(0, 1))
            ms = sorted(times)[len(times) // 2]
            by = n * (SW * 4 + 8)
            gbs = by / (ms / 1e3) / 1e9
            rows.append({"terminals": n, "bytes_per_terminal": SW * 4 + 8, "ms": round(ms, 5),
                         "gbs": round(gbs, 1), "frac_hbm": round(gbs / peak_gbs, 4) if peak_gbs else None,
                         "terminals_per_s": n / (ms / 1e3)})
            del st, res
        tr.close()
        out[name] = rows
    return out


if __name__ == "__main__":
    peak = None
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peak = json.load(open(p))["hbm_gbs"]
    print(json.dumps(sweep(peak_gbs=peak or 6548.0), indent=1))
