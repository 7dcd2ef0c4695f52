"""Benchmark: RQMC paths/s of the fused B200 path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|c5|c1|c4] [--generator NAME]

A step is one full run of the workload's replication loop (default C2:
LIBOR caplet, 20 quarterly forwards, rasrap-recursive, M = 1024
replications x N = 2^20 paths): device randomisation setup, fused generator
-> inverse normal -> Euler path -> payoff kernel, numpy-order reduction to
theta.  Multi-GPU (torchrun, one process per GPU, NCCL) is STRONG scaling,
as the reference splits a fixed M over its workers (harness.py:349-358):
rank r of W owns the contiguous replication ids distributed.shard(M, W, r),
no data-path collective, theta all-gathered once per step; the time is the
max over ranks and `value` = M x N / that time.  The gathered theta is
bit-identical for every W (`theta_sha16`).  Rank 0 prints one JSON line.

The N=1 line carries `cpu_baseline` (the oracle timed on the host cores on
`cores` replications of the same workload at full N) and `parity`: theta of
those same replication ids -- the first and the last ids of the M range, so
the last payoff batch is covered -- from the oracle against the GPU's.

--impl reference times the CPU oracle (a bit-exact C restatement of the
reference numba path, oracle/; the reference itself is Python+numba and has
no compiled artefact to run here) on the host cores with all threads, on a
bounded sample of the same workload, plus a one-thread figure (`workers_1`).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SEED = 20120224

# SURVEY 8(d) frozen FP64-slot convention (W per path / per normal)
def libor_slots(S: int) -> float:
    return 7.5 * S * S + 53.5 * S + 3


MBS_SLOTS = 97 * 360 - 2
WORKLOADS = {
    # name: (model, maturity, accrual, M, N, description)
    "c1": ("libor", 5.0, 0.25, 16, 10_000, "C1 LIBOR caplet S=20 (T=5, delta=0.25), M=16 x N=10^4"),
    "c2": ("libor", 5.0, 0.25, 1024, 2**20, "C2 LIBOR caplet S=20 (T=5, delta=0.25), M=1024 x N=2^20"),
    "c3": ("mbs", None, None, 256, 10**6, "C3 MBS 360 months, M=256 x N=10^6"),
    "c5": ("libor", 20.0, 0.25, 8192, 2**20, "C5 LIBOR caplet S=80 (T=20, delta=0.25), M=8192 x N=2^20"),
    "c4": ("stream", None, None, 1, 27_777_778,
           "C4 stream: 360-dim points with fused inverse normal, 10^10 normals per step"),
}
NORMAL_SLOTS = 36  # Phi^-1 per normal


# DRAM bytes (read + write) per path of the path kernel, from one
# `ncu --set full` capture per workload (profiles/traffic.json); the
# algorithmic traffic is the 8-byte payoff per path.
TRAFFIC_SOURCE = "profiles/traffic.json (ncu --set full: dram__bytes_read.sum + dram__bytes_write.sum)"


def _profile_entry(workload: str, gen: str) -> dict:
    try:
        tab = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        return tab[f"{workload}/{gen}"]
    except (OSError, KeyError, ValueError):
        return {}


def traffic_per_launch(workload: str, gen: str, M: int, N: int):
    bpp = _profile_entry(workload, gen).get("dram_bytes_per_path")
    if bpp is None:
        return None
    per_launch = min(M, max(1, (128 << 20) // N)) * N  # rq_estimate's replication batch
    return bpp * per_launch


def build_model(kind, maturity, accrual):
    from paper_1408_5526_b200 import models as M

    if kind == "libor":
        return M.LiborModel(M.LiborConfig(maturity=maturity, accrual=accrual))
    return M.MbsModel()


def slots_per_path(model) -> float:
    return libor_slots(model.dim) if model.name == "libor" else MBS_SLOTS


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- ours
def device_step(gen_id, model, seed, first, count, grid, theta, lib, C, _lib):
    """One workload step through the C ABI with device-resident output."""
    h = C.c_void_p()
    st = _lib.stream_ptr()
    _lib.check(lib.rq_sampler_create(C.byref(h), gen_id, model.dim, seed, first, count, st))
    ms, keep = _lib.model_struct(model)
    import numpy as np

    g = np.ascontiguousarray(grid, dtype=np.int64)
    n = C.c_int32(0)
    _lib.check(lib.rq_estimate(h, C.byref(ms), g.ctypes.data_as(C.POINTER(C.c_int64)), g.size,
                               theta.data_ptr(), C.byref(n), st))
    return h, n.value + (1 if gen_id in (0, 1, 3, 4, 7, 8) else 0), keep  # + setup kernel


def run_stream(args) -> dict:
    """Config 4: 10^10 normals of one generator (s = 360 points, Phi^-1 fused,
    consumed by a sum) per step."""
    import ctypes as C

    import numpy as np
    import torch

    from paper_1408_5526_b200 import _lib

    if int(os.environ.get("RANK", "0")) != 0:  # a one-GPU stream: other ranks idle
        return None
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count()))
    lib = _lib.lib()
    dim, npts = 360, WORKLOADS["c4"][4]
    if args.reps:
        npts = args.reps
    h = C.c_void_p()
    st = _lib.stream_ptr()
    _lib.check(lib.rq_sampler_create(C.byref(h), _lib.GEN_IDS[args.generator], dim, SEED, 0, 1,
                                     st))
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    peak, _ = _lib.fp64_peak()

    def step():
        _lib.check(lib.rq_stream_normals(h, 0, npts, out.data_ptr(), None, st))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    clocks.start()
    ms = []
    for _ in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    clk = clocks.stop()
    lib.rq_sampler_destroy(h)
    t = float(np.mean(ms))
    normals = npts * dim
    value = normals / (t * 1e-3)
    # end to end through the public API: randomisation setup, the stream,
    # the sum read back to the host, every step
    e2e_ms = []
    for it in range(1 + max(1, min(args.steps, 3))):  # iteration 0: untimed warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h2 = C.c_void_p()
        _lib.check(lib.rq_sampler_create(C.byref(h2), _lib.GEN_IDS[args.generator], dim, SEED, 0,
                                         1, st))
        _lib.check(lib.rq_stream_normals(h2, 0, npts, out.data_ptr(), None, st))
        total = float(out.item())
        lib.rq_sampler_destroy(h2)
        if it > 0:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e = {"value": normals / (float(np.mean(e2e_ms)) * 1e-3), "unit": "normals/s",
           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8,
           "api": "rq_sampler_create + rq_stream_normals (sum to host)"}
    assert math.isfinite(total)
    out = {
        "metric": "C4 normals/sec (fused inverse normal, s=360 stream)", "value": value,
        "unit": "normals/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seed 20120224, replication 0)",
        "config": {"workload": WORKLOADS["c4"][5], "generator": args.generator,
                   "points": npts, "dim": dim, "sum_check": float(out.item())},
        "roofline": {"bound": "fp64", "achieved": value * NORMAL_SLOTS / 1e12,
                     "peak": peak / 1e12, "unit": "Tslot/s (36 slots/normal)",
                     "frac": value * NORMAL_SLOTS / peak},
        "clocks": clk,
        "e2e": e2e,
        "gpu_launches": args.steps * 2,  # stream kernel + pairwise sum of the block sums
    }
    if not args.no_cpu_baseline:
        ref = run_reference_stream(argparse.Namespace(generator=args.generator, steps=1,
                                                      warmup=1))
        out["cpu_baseline"] = ref["cpu_baseline"]
    return out


def workload_config(args) -> tuple:
    """(model, M, N, desc, config dict) -- the config dict is printed by BOTH
    arms, identical, so the driver can match them."""
    kind, mat, acc, M, N, desc = WORKLOADS[args.workload]
    if args.reps:
        M = args.reps
        desc += f" [M overridden to {M}]"
    model = build_model(kind, mat, acc)
    cfg = {"workload": desc, "generator": args.generator, "M": M, "N": N, "model": kind,
           "dim": model.dim,
           "l2": "GPU arm: L2 flushed between timed steps (256 MiB write); inputs are "
                 "generated on chip"}
    return model, M, N, desc, cfg


def parity_ids(M: int, k: int):
    """The first ceil(k/2) and the last floor(k/2) replication ids of 1..M."""
    import numpy as np

    k = max(1, min(k, M))
    lo = (k + 1) // 2
    return np.unique(np.r_[np.arange(1, lo + 1), np.arange(M - (k - lo) + 1, M + 1)])


def run_ours(args) -> dict:
    import ctypes as C
    import hashlib

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1408_5526_b200 import _lib
    from paper_1408_5526_b200.distributed import shard
    from paper_1408_5526_b200.harness import estimate_replications

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_dist = "RANK" in os.environ  # launched by torchrun (any world size)
    # one GPU per rank over NCCL; with fewer GPUs than ranks (a multi-rank
    # check of this script on a one-GPU box) ranks share devices and the
    # gather runs over gloo from host copies
    ndev = torch.cuda.device_count()
    shared_dev = use_dist and ndev < world
    local = local % ndev if shared_dev else local
    torch.cuda.set_device(local)
    if use_dist:
        if shared_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    coll_dev = "cpu" if shared_dev else "cuda"
    lib = _lib.lib()
    model, M, N, desc, cfg = workload_config(args)
    gen = args.generator
    gen_id = _lib.GEN_IDS[gen]
    grid = (N,)
    # strong scaling: the fixed M split over the ranks (harness.py:349-358)
    counts = [shard(M, world, r)[1] for r in range(world)]
    off, count = shard(M, world, rank)
    first = 1 + off
    width = max(counts)
    theta = torch.zeros((width, 1), dtype=torch.float64, device="cuda")
    gathered = [torch.empty((width, 1), dtype=torch.float64, device=coll_dev)
                for _ in range(world)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    def one_step():
        h, n = None, 0
        if count:
            h, n, _ = device_step(gen_id, model, SEED, first, count, grid, theta, lib, C, _lib)
        if use_dist:  # the one collective: theta of every rank, once per step
            dist.all_gather(gathered, theta if not shared_dev else theta.cpu())
        return h, n

    def release(h):
        if h is not None:
            lib.rq_sampler_destroy(h)

    peak, peak_ms = _lib.fp64_peak()
    launches = 0
    for _ in range(args.warmup):
        h, _ = one_step()
        torch.cuda.synchronize()
        release(h)
    clocks = ClockSampler(local)
    clocks.start()
    step_ms = []
    for _ in range(args.steps):
        flush.zero_()  # L2 flushed between timed iterations
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h, n = one_step()
        b.record()
        b.synchronize()
        release(h)
        launches += n
        step_ms.append(a.elapsed_time(b))
    clk = clocks.stop()
    ms = float(np.mean(step_ms))
    ms_t = torch.tensor([ms], dtype=torch.float64, device=coll_dev)
    if use_dist:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = M * N / (ms * 1e-3)
    if use_dist:
        full = np.concatenate([g[:c].cpu().numpy() for g, c in zip(gathered, counts)])
    else:
        full = theta[:count].cpu().numpy()
    theta_sha = hashlib.sha256(np.ascontiguousarray(full, dtype=np.float64).tobytes()).hexdigest()

    # kernel share: one extra (untimed) step with per-kernel CUDA events
    _lib.stats_reset(timing=True)
    h, _ = one_step()
    torch.cuda.synchronize()
    release(h)
    ks = _lib.stats_get()
    _lib.stats_reset(timing=False)
    W = slots_per_path(model)
    achieved = count * N * W / max(ks["paths_ms"] * 1e-3, 1e-12)  # this GPU, slots/s

    # end to end through the host API: host in, theta to host every step
    e2e_ms = []
    _lib.stats_reset(timing=False)
    for k in range(max(1, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        if count:
            estimate_replications(gen, model, SEED, first, count, grid)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    tr = _lib.stats_get()
    ne = len(e2e_ms)
    e2e_t = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=coll_dev)
    if use_dist:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    e2e_value = M * N / (float(e2e_t.item()) * 1e-3)

    out = None
    if rank == 0:
        out = {
            "metric": "RQMC paths/sec (LIBOR caplet, MBS) at 1/2/4/8 B200; % FP64 pipe peak",
            "value": value,
            "unit": "paths/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seed 20120224, replication ids 1..M, packaged 2012-02-24 "
                    "Treasury curve)",
            "config": cfg,
            "parallelism": f"replication-sharded x{world}: fixed M={M} split, "
                           f"{count} replications on rank 0 (theta all-gathered once per step"
                           + ((" over gloo, ranks sharing " + str(ndev) + " GPU(s))"
                               if shared_dev else " over NCCL)") if use_dist else ")"),
            "M_per_rank": counts,
            "theta_sha16": theta_sha[:16],
            "roofline": {
                "bound": "fp64",
                "kernel": "k_paths_* (fused generator + inverse normal + path + payoff)",
                "achieved": achieved / 1e12,
                "peak": peak / 1e12,
                "unit": "Tslot/s (FP64 pipe slots, SURVEY 8(d) convention)",
                "frac": achieved / peak,
                "slots_per_path": W,
                "peak_source": "measured on this GPU by rq_fp64_peak (DFMA probe, burst)",
                "paths_kernel_share": ks["paths_ms"] / max(ks["paths_ms"] + ks["reduce_ms"]
                                                           + ks["setup_ms"], 1e-9),
                "kernel_ms": {"setup": ks["setup_ms"], "paths": ks["paths_ms"],
                              "reduce": ks["reduce_ms"]},
                "traffic": traffic_per_launch(args.workload, gen, count, N),
                "traffic_source": TRAFFIC_SOURCE,
                "ncu_fp64_pipe_pct": _profile_entry(args.workload, gen).get("fp64_pipe_pct"),
            },
            "e2e": {"value": e2e_value, "unit": "paths/s",
                    "h2d_bytes_per_step": tr["h2d"] // ne, "d2h_bytes_per_step": tr["d2h"] // ne,
                    "api": "rq_run_replications (host in / theta to host)"},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if not args.no_cpu_baseline and world == 1:  # the CPU baseline: N=1 runs only
            cb, par = cpu_baseline(model, gen, M, N, full[:, 0])
            out["cpu_baseline"] = cb
            out["parity"] = par
        if args.workload == "c2" and not use_dist and not args.reps:
            out["comparison"] = generator_comparison(model, M, N)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return out


def generator_comparison(model, M: int, N: int) -> dict:
    """Config 2's comparison (BASELINE configs[1]): random-start Halton vs
    Philox MC vs scrambled Sobol' on the same caplet, M x N, through the
    host API.  Standard error SE = std(theta) / sqrt(M); the reference's
    efficiency column is std x seconds per replication (harness.py:364-385);
    variance reduction = (SE_philox / SE)^2 at equal N."""
    import numpy as np

    from paper_1408_5526_b200.harness import estimate_replications

    res = {}
    for g in ("rasrap-recursive", "philox", "sobol-gray"):
        estimate_replications(g, model, SEED, 1, 2, (N,))  # warm
        t0 = time.perf_counter()
        th = estimate_replications(g, model, SEED, 1, M, (N,))[:, 0]
        sec = time.perf_counter() - t0
        std = float(np.std(th, ddof=1))
        res[g] = {"paths_per_s": M * N / sec, "mean": float(th.mean()),
                  "std_error": std / math.sqrt(M), "efficiency_std_x_s": std * sec / M,
                  "std_error_per_s": std / math.sqrt(M) / sec}
    base = res["philox"]["std_error"]
    for g in res:
        res[g]["variance_reduction_vs_philox"] = (base / res[g]["std_error"]) ** 2
    return {"workload": f"LIBOR S={model.dim}, M={M} x N={N}, seed {SEED}", "generators": res}


# ---------------------------------------------------------------- reference arm
def _sobol_v(model, gen):
    if not gen.startswith("sobol"):
        return None
    from paper_1408_5526_b200.tables import sobol_directions

    return sobol_directions(model.dim)


def cpu_theta(model, gen, ids, N, threads):
    """(theta[ids], seconds): the oracle on replication ids (runs of
    consecutive ids), `threads` host threads, each owning whole replications
    (harness.py:349-358)."""
    import numpy as np

    from oracle import oracle as O

    runs = np.split(ids, np.where(np.diff(ids) != 1)[0] + 1)
    # the runs go concurrently (the ctypes call releases the GIL), the host
    # threads split in proportion to their replications, so every thread
    # owns whole replications as in one run
    share = [max(1, round(threads * len(r) / len(ids))) for r in runs]
    th = [None] * len(runs)
    sob = _sobol_v(model, gen)

    def go(k):
        r = runs[k]
        th[k] = O.run_replications(gen, model, SEED, int(r[0]), len(r), (N,), threads=share[k],
                                   sobol_v=sob)[:, 0]

    t0 = time.perf_counter()
    pool = [threading.Thread(target=go, args=(k,)) for k in range(len(runs))]
    for t in pool:
        t.start()
    for t in pool:
        t.join()
    return np.concatenate(th), time.perf_counter() - t0


THETA_RTOL = 1e-12  # north_star: per-replication estimates within ~1e-12 (FP64)


def cpu_baseline(model, gen, M, N, theta_gpu) -> tuple[dict, dict]:
    """The oracle on `cores` replications at full N -- the first and the last
    ids of 1..M -- timed on the host cores, and their theta against the
    GPU's (theta_gpu[m - 1] for id m)."""
    import numpy as np

    from oracle import oracle as O

    cores = O.host_cores()
    ids = parity_ids(M, cores)
    ref, sec = cpu_theta(model, gen, ids, N, cores)
    got = theta_gpu[ids - 1]
    rel = float(np.max(np.abs(got / ref - 1.0)))
    span = f"{ids[0]}-{ids[(len(ids) + 1) // 2 - 1]},{ids[(len(ids) + 1) // 2]}-{ids[-1]}" \
        if len(ids) > 1 else str(ids[0])
    cb = {"value": len(ids) * N / sec, "unit": "paths/s", "cores": cores, "kind": "port",
          "sample": f"{len(ids)} replications (ids {span}) x N={N} of the same workload "
                    f"({gen}), oracle/rqmc_oracle.c (bit-exact C restatement of the "
                    f"reference numba path), {cores} threads"}
    par = {"reps": int(len(ids)), "ids": span, "max_rel_err": rel, "tol": THETA_RTOL,
           "ok": bool(rel <= THETA_RTOL), "bit_exact_reps": int(np.sum(got == ref))}
    return cb, par


def cpu_stream_normals(gen: str, first: int, count: int, dim: int = 360) -> float:
    """Config 4 on the host: the oracle's points first..first+count-1 of
    replication 0 (the reference layouts) through the reference Phi^-1,
    summed.  Returns the sum."""
    import numpy as np

    from oracle import oracle as O

    idx = np.arange(first, first + count, dtype=np.int64)
    if gen == "philox":
        u = O.philox_words(O.derive_key(SEED, 3, 0), idx, dim) * 2.0**-32 + 2.0**-33
    elif gen == "sfc64":
        u = O.sfc64_uniforms(SEED, 0, idx, dim)
    elif gen.startswith("sobol"):
        from paper_1408_5526_b200.tables import sobol_directions

        gv, sh = O.sobol_scramble(sobol_directions(dim), O.derive_key(SEED, 5, 0), 0)
        ii = idx ^ (idx >> 1) if gen == "sobol-gray" else idx
        u = O.sobol_counter_words(gv, sh, ii) * 2.0**-32
    else:  # rasrap: the counter form at the indices (the recursive form equals it to 1e-12)
        u = O.rasrap_counter(dim, O.derive_key(SEED, 4, 0), idx)
    return float(O.inv_normal(u).sum())


def run_reference_stream(args) -> dict:
    """--impl reference --workload c4: the same normals stream on the host
    cores (threads over point blocks; the ctypes calls release the GIL)."""
    from oracle import oracle as O

    cores = O.host_cores()
    dim, pts = 360, 200_000  # bounded sample: 7.2e7 normals per step
    blk = (pts + cores - 1) // cores

    def step():
        th = [threading.Thread(target=cpu_stream_normals,
                               args=(args.generator, k * blk, min(blk, pts - k * blk), dim))
              for k in range(cores) if k * blk < pts]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        return pts * dim / (time.perf_counter() - t0)

    for _ in range(args.warmup):
        cpu_stream_normals(args.generator, 0, 1000, dim)
    v = float(statistics.median([step() for _ in range(args.steps)]))
    return {
        "metric": "C4 normals/sec (fused inverse normal, s=360 stream)", "impl": "reference",
        "value": v, "unit": "normals/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pts * dim / v * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seed 20120224, replication 0)",
        "config": {"workload": WORKLOADS["c4"][5], "generator": args.generator, "dim": dim},
        "cpu_baseline": {"value": v, "unit": "normals/s", "cores": cores, "kind": "port",
                         "sample": f"{pts} points x {dim} dims per step, {args.generator} "
                                   f"(oracle generator + reference Phi^-1), {cores} threads"},
        "e2e": {"value": v, "unit": "normals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference(args) -> dict | None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    if args.workload == "c4":
        return run_reference_stream(args)
    from oracle import oracle as O

    model, M, N, desc, cfg = workload_config(args)
    gen = args.generator
    cores = O.host_cores()
    # bounded per-step sample: `cores` whole replications (C2: full N; the
    # long-path workloads at N/16 -- paths/s is independent of N)
    n = N if model.dim <= 20 else max(8192, N // 16)
    ids = parity_ids(M, cores)
    for _ in range(args.warmup):
        cpu_theta(model, gen, ids[:2], 8192, cores)
    rates = []
    for _ in range(args.steps):
        _, sec = cpu_theta(model, gen, ids, n, cores)
        rates.append(len(ids) * n / sec)
    v = float(statistics.median(rates))
    _, sec1 = cpu_theta(model, gen, ids[:1], n, 1)  # workers = 1
    samp = (f"{len(ids)} replications x N={n} per step (of M={M} x N={N}), {gen}, "
            f"{cores} threads (oracle/rqmc_oracle.c, bit-exact restatement of the reference "
            f"numba kernels)")
    return {
        "metric": "RQMC paths/sec (LIBOR caplet, MBS) at 1/2/4/8 B200; % FP64 pipe peak",
        "impl": "reference",
        "value": v,
        "unit": "paths/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": len(ids) * n / v * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seed 20120224, replication ids 1..M, packaged 2012-02-24 "
                "Treasury curve)",
        "config": cfg,
        "cpu_baseline": {"value": v, "unit": "paths/s", "cores": cores, "kind": "port",
                         "sample": samp},
        "workers_1": {"value": n / sec1, "unit": "paths/s", "cores": 1,
                      "sample": f"1 replication x N={n}, 1 thread"},
        "e2e": {"value": v, "unit": "paths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--generator", default="rasrap-recursive")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reps", type=int, default=0,
                    help="override M (total replications, split over the ranks; for c4 the point count) for quick sub-runs")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.workload == "c4" and args.impl == "ours":
        out = run_stream(args)
    else:
        out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
