#!/usr/bin/env python
"""bench.py — GFlowNet training throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): hypergrid 20^4, detailed balance, MLP 2x256,
65536 trajectories per GPU per iteration (weak scaling: N GPUs train on N x 65536
trajectories per iteration, one NCCL all-reduce of the gradient per iteration).
A "step" is one full training iteration: forward rollout (sampling from the current
policy), loss + gradient, all-reduce, Adam — train_scenario's loop body
(proj/src/train.cpp:224-229), entirely on the device.

  value  trajectories/s with everything resident, timed with CUDA events on the engine
         stream, max over ranks.
  e2e    the same through the public C ABI call per iteration (gfnx_iteration) with the
         loss and the batch's terminal states / lengths / log-rewards copied to host
         buffers every iteration (what the reference loop hands to its FIFO buffer,
         train.cpp:231), timed on the host clock, max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one process per GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import threading
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = "hypergrid_db_b65536"
PER_GPU_BATCH = 65536
METRIC = "trajectories/sec (train iters/sec in config) — hypergrid 20^4 DB, B=65536/GPU"
UNIT = "trajectories/s"
# secondary BASELINE configs measured after the headline (device-timed, resident inputs)
SECONDARY = {
    "hypergrid_subtb_b65536": dict(batch=65536, desc="hypergrid 20^4 SubTB (lambda 0.9), B=65536, MLP 2x256"),
    "bitseq_tb_b16384": dict(batch=16384, desc="bitseq n=120 k=8 NAR TB, MLP 2x256"),
    "bitseq_ar_tb_b16384": dict(batch=16384, desc="bitseq n=120 k=8 autoregressive (fixed) TB, MLP 2x256"),
    "ising_tb_b32768": dict(batch=32768, desc="Ising 10x10 TB, MLP 4x256"),
    "hypergrid_tb_b16": dict(batch=16, desc="hypergrid 20^4 TB, B=16, MLP 2x256"),
    "dag_mdb_b8192": dict(batch=8192, desc="DAG d=5 BGe MDB, MLP 2x128"),
    # the headline workload in deterministic mode (static per-CTA ranges, bit-identical reruns)
    "hypergrid_db_b65536_det": dict(batch=65536, config="hypergrid_db_b65536", det=1,
                                    desc="hypergrid 20^4 DB, B=65536, MLP 2x256, deterministic=1"),
    # EB-GFN (run_eb_gfn): the paper's Ising setting (PAPER Table 1: N = 10, TB, B = 256, MLP
    # 4x256, 26.4 it/s for JAX gfnx on a GPU); k = D back-and-forth steps, data batch 256
    "eb_gfn_ising10_b256": dict(batch=256, eb=True,
                                desc="EB-GFN Ising 10x10, TB sampler B=256 MLP 4x256 (bf16 lockstep), "
                                     "k=100, data batch 256; it/s (PAPER: 26.4 it/s, JAX gfnx)"),
}


def secondary_runs(names, steps, warmup, local):
    from paper_2511_16592_b200 import abi, engine
    out = {}
    for name in names:
        spec = SECONDARY[name]
        if spec.get("eb"):
            out[name] = eb_leg(spec, steps, warmup, local)
            continue
        try:
            e, t = abi.config(spec.get("config", name), batch=spec["batch"])
            t.iterations = 1_000_000
            t.deterministic = spec.get("det", 0)
            tr = engine.Trainer(e, t, device=local)
            tr.run(0, warmup)
            tr.synchronize()
            tr.profile(True)
            tr.event_record(0)
            tr.run(warmup, steps)
            tr.event_record(1)
            tr.synchronize()
            ms = tr.event_elapsed(0, 1)
            prof = tr.profile_read()
            out[name] = {"workload": spec["desc"], "trajectories_per_s": spec["batch"] * steps / (ms / 1e3),
                         "iters_per_s": steps / (ms / 1e3), "ms_per_iter": ms / steps,
                         "kernels_ms_per_iter": {k: round(v[0] / steps, 4) for k, v in prof.items()}}
            tr.close()
        except Exception as ex:  # reported, never fatal
            out[name] = {"error": str(ex)[:300]}
    return out


def eb_leg(spec, steps, warmup, local):
    """EB-GFN iterations/s on the device (gfnx_eb_run: mixture rollout, train step, k-step
    back-and-forth proposals, MH, CD update per iteration), CUDA events on the engine stream."""
    from paper_2511_16592_b200 import abi, engine
    try:
        e = abi.env_desc(abi.ISING, is_side=10, is_sigma=0.2)
        t = abi.train_desc(abi.ISING, batch=spec["batch"], iterations=1_000_000)
        tr = engine.Trainer(e, t, device=local)
        tr.eb_init(engine.eb_desc(data_batch=spec["batch"]))
        tr.eb_run(0, warmup)
        tr.synchronize()
        tr.event_record(0)
        m = tr.eb_run(warmup, steps)
        tr.event_record(1)
        tr.synchronize()
        ms = tr.event_elapsed(0, 1)
        _, _, init_nlr = tr.eb_coupling()
        tr.close()
        return {"workload": spec["desc"], "iters_per_s": steps / (ms / 1e3), "ms_per_iter": ms / steps,
                "trajectories_per_s": spec["batch"] * steps / (ms / 1e3),
                "neg_log_rmse": [round(init_nlr, 4), round(float(m[-1, 2]), 4)]}
    except Exception as ex:  # reported, never fatal
        return {"error": str(ex)[:300]}


STEADY_CKPT = os.path.join(ROOT, "profiles", "hypergrid_db_converged.ckpt")


def steady_state_leg(e, t, local, W, K):
    """The headline workload from a CONVERGED policy (GFNCKPT1 checkpoint trained on the device
    by profiles/make_converged_ckpt.py): the trajectory length under the target policy is
    ~39 steps instead of ~5 at initialisation, so traj/s drops and rows/s is the
    comparable rate. Device-timed like the headline (CUDA events on the engine stream)."""
    from paper_2511_16592_b200 import engine
    if not os.path.exists(STEADY_CKPT):
        return {"error": "profiles/hypergrid_db_converged.ckpt missing"}
    tr = engine.Trainer(e, t, device=local)
    step = tr.load_checkpoint(STEADY_CKPT)
    _, tv0 = tr.exact_terminal_marginal(20 ** 4)
    tr.run(step, W)
    r0 = tr.counters()[0]
    tr.synchronize()
    tr.event_record(0)
    tr.run(step + W, K)
    tr.event_record(1)
    tr.synchronize()
    ms = tr.event_elapsed(0, 1)
    rows = tr.counters()[0] - r0
    B = t.batch_size
    out = {"checkpoint": os.path.relpath(STEADY_CKPT, ROOT), "checkpoint_step": step, "tv_exact_at_load": tv0,
           "trajectories_per_s": B * K / (ms / 1e3), "rows_per_s": rows / (ms / 1e3),
           "iters_per_s": K / (ms / 1e3), "ms_per_iter": ms / K, "mean_traj_len": rows / (B * K),
           "iteration_tensor_frac": 8.0 * m_row(256, 5) * rows / (ms / 1e3) / 1e12 / measured_peaks()[1]}
    tr.close()
    return out


def reward_sweep_leg(local, hbm):
    """batched terminal-reward kernels over 2^16..2^26 terminals."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("reward_sweep", os.path.join(ROOT, "profiles", "reward_sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    res = mod.sweep(sizes=(1 << 16, 1 << 20, 1 << 24, 1 << 26), reps=10, device=local, peak_gbs=hbm)
    return {k: [{"terminals": r["terminals"], "gbs": r["gbs"], "frac_hbm": r["frac_hbm"]} for r in v]
            for k, v in res.items()}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Comm:
    """Control-plane collectives over gloo (the data-plane all-reduce is NCCL in libgfnx)."""

    def __init__(self, world, rank):
        self.world, self.rank = world, rank
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group("gloo", rank=rank, world_size=world)
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def bcast_bytes(self, b: bytes | None) -> bytes:
        if not self.dist:
            return b
        obj = [b]
        self.dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def close(self):
        if self.dist:
            self.dist.destroy_process_group()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def start(self):
        """Launch the sampler and wait (<= 5 s) for its first line: nvidia-smi needs ~0.5-1 s
        to start, longer than a short timed region."""
        self.lines, self.i0 = [], 0
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.gpu)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
            return

        def pump():
            for line in self.p.stdout:
                self.lines.append(line)

        self.t = threading.Thread(target=pump, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.lines and time.time() - t0 < 5.0 and self.p.poll() is None:
            time.sleep(0.02)
        self.i0 = len(self.lines)  # samples from here on fall inside the measured region

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0 = time.time()  # at least one sample taken after the region started
        while len(self.lines) <= self.i0 and time.time() - t0 < 1.0 and self.p.poll() is None:
            time.sleep(0.02)
        self.p.terminate()
        try:
            self.p.wait(timeout=10)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.t.join(timeout=5)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines[self.i0:]:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def m_row(H, A, flow=True):
    """SURVEY §8(d) MACs per state row of the layers after the one-hot layer 1 (a row gather
    of W1, counted in bytes): hidden H x H plus the heads the objective uses (fwd [+ flow])."""
    return H * H + H * (A + (1 if flow else 0))


def kernel_work(name, rows, iters, H, A, n_params, batch=0, SW=1):
    """SURVEY §8(d) ALGORITHMIC FLOPs and HBM bytes of `iters` launches of `name` over `rows`
    real state rows in total (not the design's own materialisation):
      tensor FLOPs   2 * M_row per row for each of the rollout forward, the dgrad and the wgrad
                     (the training forward is fused into the rollout; §8(d) counts 8 M_row per
                     row for the whole iteration: rollout fwd + training fwd + dgrad + wgrad)
      HBM bytes      (i) 23 B per live (b, t) for the rollout/step (5 bf16 logits + state r/w +
                     action + log-prob), (iv) 28 B per parameter for Adam, the loss record once"""
    R = rows
    M = m_row(H, A)
    if name in ("k_fast_rollout", "k_fast_fwd"):
        return 2.0 * M * R, (A * 2 + 2 * 4 + 1 + 4) * R + batch * (4 + 8 + 4 * SW)
    if name in ("k_fast_bwd", "k_fast_wgrad"):
        return 2.0 * M * R, 0.0
    if name == "k_row_stats":
        return 0.0, R * ((A + 1) * 4 + 4 * 4)
    if name == "k_fast_loss":
        return 0.0, R * (4 * 4 + 4 + 2) + batch * 16
    if name == "k_reduce":
        return 0.0, 2 * n_params * 4 * iters
    if name == "k_fast_adam":
        return 0.0, 28.0 * n_params * iters
    return 0.0, 0.0


def cpu_reference_sample(steps: int, warmup: int, procs: int, batch: int):
    """The reference's own run_bench (train.cpp:294-334) via oracle/_ref, one process per
    host core (the reference is single-threaded), hypergrid 20^4 DB at `batch` trajectories."""
    import multiprocessing as mp
    kv = {"env.dim": 4, "env.side": 20, "objective.name": "db", "train.batch_size": batch,
          "bench.repeats": 1, "bench.iters": steps, "bench.warmup": warmup, "eval.metrics": "",
          "seed": 0}
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.starmap(_ref_worker, [(kv, i) for i in range(procs)])
    its = [r for r in res if r is not None]
    return its


def _ref_worker(kv, i):
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    kv = dict(kv)
    kv["seed"] = i
    kind = "fast" if O.ref_available("fast") else "port"
    mean, _ = O.ref_run_bench("hypergrid", kv, kind=kind)
    return mean


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle as O
    procs = max(1, min(os.cpu_count() or 1, 64))
    batch = 32
    t0 = time.perf_counter()
    its = cpu_reference_sample(args.steps, args.warmup, procs, batch)
    wall = time.perf_counter() - t0
    value = float(sum(its) * batch)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * batch * procs / value if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (environment-generated trajectories)",
        "config": {"workload": CONFIG, "env": "hypergrid d=4 H=20", "objective": "db",
                   "mlp": "2x256", "global_batch": batch * procs,
                   "sample": f"{procs} processes x B={batch} (distinct seeds); the workload's "
                             f"B={PER_GPU_BATCH * args.gpus} per iteration is infeasible on CPU "
                             f"(~10^3 s / iteration, >100 GB of tape), per-trajectory cost is ~flat in B",
                   "build": "reference sources, g++ -O3 -march=x86-64-v3 (FMA on; the shipped CMake "
                            "flags use -march=native, not portable to the GPU box's host)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs,
                         "kind": "reference" if O.ref_available("fast") else "port",
                         "sample": f"{procs} processes x reference run_bench(hypergrid 20^4 DB, "
                                   f"B={batch}, iters={args.steps}, warmup={args.warmup}); "
                                   f"wall {wall:.1f}s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def cpu_baseline_leg():
    """Single-core reference timing on a bounded sample (~10-30 s), rank 0 at N=1 only."""
    from oracle import oracle as O
    batch, iters = 128, 6
    kind = "fast" if O.ref_available("fast") else ("port" if O.ref_available("port") else None)
    t0 = time.perf_counter()
    if kind is not None:
        kv = {"env.dim": 4, "env.side": 20, "objective.name": "db", "train.batch_size": batch,
              "bench.repeats": 1, "bench.iters": iters, "bench.warmup": 1, "eval.metrics": "",
              "seed": 0}
        its, _ = O.ref_run_bench("hypergrid", kv, kind=kind)
        return {"value": its * batch, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"reference run_bench (oracle/_ref, {kind} build), hypergrid 20^4 DB, "
                          f"B={batch}, 1 warmup + {iters} timed iterations, "
                          f"{time.perf_counter() - t0:.1f}s wall"}
    from paper_2511_16592_b200 import abi
    e, t = abi.config(CONFIG, batch=batch)
    o = O.Oracle(e, t)
    o.iteration(0)
    t1 = time.perf_counter()
    for it in range(1, 1 + iters):
        o.iteration(it)
    dt = time.perf_counter() - t1
    return {"value": batch * iters / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle restatement, hypergrid 20^4 DB, B={batch}, {iters} iterations"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=PER_GPU_BATCH, help="trajectories per GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-steady", action="store_true", help="skip the converged-checkpoint leg")
    ap.add_argument("--no-sweep", action="store_true", help="skip the reward-kernel B sweep")
    ap.add_argument("--secondary", default="hypergrid_subtb_b65536,bitseq_tb_b16384,bitseq_ar_tb_b16384,"
                                           "ising_tb_b32768,hypergrid_tb_b16,dag_mdb_b8192,hypergrid_db_b65536_det,"
                                           "eb_gfn_ising10_b256",
                    help="comma list of secondary configs (device-timed), '' to skip")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    from paper_2511_16592_b200 import abi, engine
    comm = Comm(world, rank)
    e, t = abi.config(CONFIG, batch=args.batch * world)
    t.iterations = 1_000_000
    nccl_id = engine.nccl_unique_id() if (world > 1 and rank == 0) else None
    nccl_id = comm.bcast_bytes(nccl_id) if world > 1 else None
    tr = engine.Trainer(e, t, device=local, rank=rank, world=world, nccl_id=nccl_id)
    W, K = max(args.warmup, 3), args.steps
    tr.run(0, W - 2)
    for i in (W - 2, W - 1):  # the last two warm-up iterations go through the e2e path (pinned slots)
        tr.iteration_async(i, i % 2)
    tr.slot_wait(W % 2)
    tr.slot_wait((W + 1) % 2)
    tr.synchronize()

    # ---- end to end through the C ABI: per iteration, results copied to pinned host
    # memory (gfnx_iteration_async + gfnx_slot_wait, two slots in flight) and consumed.
    # Runs iterations W..W+K-1 first; the policy + Adam state are then restored so the
    # device-timed region below replays exactly the same K iterations (same trajectories).
    e2e = None
    snap = (tr.params(), tr.adam_state())
    clocks = ClockSampler(local)
    clocks.start()
    if not args.no_e2e:
        comm.barrier()
        tr.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        sink = 0.0
        for i in range(K):
            tr.iteration_async(W + i, i % 2)
            if i > 0:
                _, loss, res = tr.slot_wait((i - 1) % 2)
                sink += loss + float(res["log_rewards"][0])
                d2h = 8 + sum(v.nbytes for v in res.values())
        _, loss, res = tr.slot_wait((K - 1) % 2)
        tr.synchronize()
        dt = comm.max(time.perf_counter() - t0)
        e2e = {"value": args.batch * world * K / dt, "unit": UNIT,
               "h2d_bytes_per_step": 24, "d2h_bytes_per_step": d2h,
               "note": "gfnx_iteration_async per step: h2d = iteration index, lr, eps (kernel "
                       "arguments); d2h = loss + lengths/log-rewards/terminal states into pinned "
                       "host memory, consumed by the host every step; host wall clock"}
    tr.set_params(*snap[0])
    tr.set_adam_state(*snap[1])
    tr.synchronize()

    # ---- device-timed region: everything resident, CUDA events on the engine stream; only
    # the rollout kernel is bracketed (its duration feeds the roofline), the full per-kernel
    # breakdown comes from a replay of the same iterations below
    launches0 = tr.kernel_launches()
    rows0, rolls0 = tr.counters()[:2]
    tr.profile(2)
    comm.barrier()
    tr.synchronize()
    tr.event_record(0)
    tr.run(W, K)
    tr.event_record(1)
    tr.synchronize()
    comm.barrier()
    ms = comm.max(tr.event_elapsed(0, 1))
    prof_timed = tr.profile_read()
    tr.profile(False)
    launches = tr.kernel_launches() - launches0
    rows1, rolls1 = tr.counters()[:2]
    rows = rows1 - rows0
    value = args.batch * world * K / (ms / 1e3)
    # per-kernel breakdown: replay of the same K iterations with every launch bracketed
    tr.set_params(*snap[0])
    tr.set_adam_state(*snap[1])
    tr.synchronize()
    tr.profile(True)
    tr.run(W, K)
    tr.synchronize()
    prof = tr.profile_read()
    tr.profile(False)
    prof.update(prof_timed)  # the rollout's own time from the timed region

    cl = clocks.stop()

    # ---- roofline of the dominant kernel (SURVEY §8(d) algorithmic work / measured time)
    hbm, tens, peak_kind = measured_peaks()
    H, A = 256, 5
    dom, dom_ms = max(prof.items(), key=lambda kv: kv[1][0]) if prof else (None, (0, 0))
    roof = None
    kernels = {}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f)
    for name, (tot_ms, cnt) in prof.items():
        fl, by = kernel_work(name, rows, K, H, A, tr.n_params, batch=args.batch * K)
        sec = tot_ms / 1e3
        kernels[name] = {"ms_total": round(tot_ms, 4), "launches": cnt, "share_of_step": round(tot_ms / ms, 4),
                         "tflops": fl / sec / 1e12 if sec and fl else None,
                         "gbs": by / sec / 1e9 if sec and by else None}
    if dom:
        fl, by = kernel_work(dom, rows, K, H, A, tr.n_params, batch=args.batch * K)
        sec = dom_ms[0] / 1e3
        per = dom_ms[1]
        if fl > 0:  # GEMM-dominated kernels: the tensor roof (bf16, sustained)
            roof = {"kernel": dom, "bound": "tensor", "achieved": fl / sec / 1e12, "peak": tens,
                    "unit": "TFLOP/s", "frac": fl / sec / 1e12 / tens}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": by / sec / 1e9, "peak": hbm,
                    "unit": "GB/s", "frac": by / sec / 1e9 / hbm}
        roof["peak_source"] = peak_kind + " (MEASURED_PEAKS.json: bf16 sustained, HBM copy)"
        roof["share_of_step"] = dom_ms[0] / ms if ms else None
        roof["algorithmic_per_launch"] = {"flops": fl / per if per else None, "bytes_8d_i": by / per if per else None,
                                          "rows": rows / K, "flops_per_row": 2 * m_row(H, A)}
        roof["hbm_frac_of_8d_i_bytes"] = by / sec / 1e9 / hbm if sec else None
        tk = (traffic or {}).get(dom) or (traffic or {}).get(dom + "_ts")  # H = 256: k_fast_rollout_ts
        if tk:  # ncu --set full of a launch of the same command (profiles/ncu_capture.py)
            roof["traffic"] = tk["dram_bytes"]
            roof["traffic_per_row"] = tk["dram_bytes"] / max(tk["rows"], 1)
            roof["traffic_source"] = tk.get("source")
        else:
            roof["traffic"] = None
    # the whole iteration against the tensor roof: 8 M_row FLOPs per real row
    it_flops = 8.0 * m_row(H, A) * rows
    iteration_roof = {"flops_per_iter": it_flops / K, "achieved_tflops": it_flops / (ms / 1e3) / 1e12,
                      "peak": tens, "frac": it_flops / (ms / 1e3) / 1e12 / tens}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_leg()
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"failed: {ex}"}

    steady = None
    if rank == 0 and world == 1 and not args.no_steady:
        try:
            steady = steady_state_leg(e, t, local, W, K)
        except Exception as ex:  # reported, never fatal
            steady = {"error": str(ex)[:300]}
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        try:
            sweep = reward_sweep_leg(local, hbm)
        except Exception as ex:  # reported, never fatal
            sweep = {"error": str(ex)[:300]}

    secondary = None
    if rank == 0 and world == 1 and args.secondary:
        secondary = secondary_runs([x for x in args.secondary.split(",") if x], max(3, K // 5), 2, local)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (trajectories generated on device by the environment)",
            "config": {"workload": CONFIG, "env": "hypergrid d=4 H=20", "objective": "db",
                       "mlp": "2x256", "batch_per_gpu": args.batch,
                       "global_batch": args.batch * world, "parallelism": f"dp{world}",
                       "train_iters_per_sec": K / (ms / 1e3),
                       "mean_traj_len": rows / (args.batch * K) if K else None,
                       "l2": "working set > L2 (bf16 activation images ~2 KB per state row)"},
            "rows_per_s": rows / (ms / 1e3), "iteration_roofline": iteration_roof,
            "e2e": e2e, "gpu_launches": launches, "roofline": roof, "kernels": kernels,
            "steady_state": steady, "reward_sweep": sweep,
            "cpu_baseline": cpu, "clocks": cl, "secondary": secondary,
        }
        print(json.dumps(line))
    tr.close()
    comm.close()


if __name__ == "__main__":
    main()
