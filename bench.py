#!/usr/bin/env python
"""bench.py -- AZ solves/s on BASELINE config 2 (1-D, N = 2^20 centres, L = 2, 64 RHS, R = 64
probes, tol 1e-12) on B200, with the roofline of the dominant kernel and the CPU oracle beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One "step" = one az_solve (Alg. 1: b' = (I - A Z*) b, the 64-probe sketch
(A - A Z* A) Omega, TSQR + truncated SVD, x2 = Omega y, step 2 x = x2 + Z*(b - A x2)) over the
config's whole RHS batch, inputs resident in HBM.  Multi-GPU (torchrun): ONE solve sharded over the
ranks by az_solve_sharded (probe / RHS column shards, NCCL all-to-all re-block, fixed 8-leaf TSQR
tree; strong scaling); --replicas times independent per-rank solves (weak
scaling) instead; the time is the max over ranks.  The reference arm (--impl reference) times the CPU oracle (oracle/, the
paper's algorithm with numpy FFTs) on a bounded sample of the same workload, scaled to one solve.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2308_14490_b200 import inputs as I  # noqa: E402

METRIC = "AZ solves/s"
UNIT = "solves/s"
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # SMs x FP64 FMA/clk/SM x 2 x max clock


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ------------------------------------------------------------------------------------------
# algorithmic bytes / flops per unit (per complex vector PAIR for the pass kernels), DESIGN.md
# "Algorithmic bytes per kernel".  n = coefficient length, L = fine length, M = rows.
# ------------------------------------------------------------------------------------------
def kernel_model(name, cfg, M, k_cols, k1=None, kept=False, split=False):
    n = cfg.N
    L = cfg.N * cfg.s ** cfg.dim
    C = 16  # bytes per complex128
    # 1-D intervals: the mask is one run of the grid, so no row-map / mask bytes are read
    pos_b, mask_b = (0, 0) if cfg.dim == 1 else (4, 1)
    # kept: the four-step narrow solve stores Omega (probe pass) for step 2 and takes the Z* parts of
    # the b' and sketch chains to the coefficient side (row passes write them, two column passes finish)
    kw_om, kw_z = (0, C * n) if kept else (0, 0)
    kw_aom = 0
    hbm = {
        "1f_cols_in_coef": C * n + kw_om,              # probes generated on chip; write spectrum (+ Omega)
        "1f_rows_expand_keep": 2 * C * n + C * L,
        "1f_rows_expand": C * n + C * L,
        "1f_rows_expand_probe": C * n + C * L,         # spectral probes drawn in the row: write v^ and the fine grid
        "1f_rows_probe_z": C * n,                      # spectral probes -> IFFT_N2 -> Z2 (explicit Omega)
        "1f_cols_fine_mask": 2 * C * L + mask_b * L + kw_aom,   # fine grid in/out, mask (1 B) (+ A Omega rows)
        "1f_rows_step1": 2 * C * L + C * n + 8 * n + kw_z,    # fine grid in/out, v^ and zinv in (+ Z* part)
        "1f_rows_resid": 2 * C * L + 8 * n + kw_z,
        "1f_rows_zstar": C * L + C * n + 8 * n,
        "1f_cols_out_gather": C * L + pos_b * L + 2 * 8 * M,   # fine grid + row map in, 2 columns out
        "1f_cols_out_resid": C * L + pos_b * L + 4 * 8 * M,
        "1f_cols_in_rows": pos_b * L + 2 * 8 * M + C * L,
        "1f_cols_out_coef": C * n + 2 * 8 * n,
        "1f_cols_out_coef_add": C * n + 4 * 8 * n,             # spectrum + x2 in, x out
        "1f_cols_resid_mid": 2 * C * L + 2 * 8 * M,            # fine grid in/out, b rows in
        "1f_cols_out_z": C * n + 2 * 8 * n,                    # Z* b: spectrum in, 2 columns out
    }
    if name in hbm:
        return "hbm", hbm[name]
    if name == "tsqr_leaf":
        # Householder on [S | b'] triangularising the k1 probe columns: per row and reflector j a
        # dot product and an axpy over the k - j - 1 trailing columns (4 flops each) plus the norm.
        # Split leaf (single probe block, az_qr.cu): this pass holds the k1 probe columns only.
        k1 = k_cols if k1 is None else k1
        kk = k1 if split else k_cols
        return "alu", float(sum(4 * (kk - j - 1) + 2 for j in range(k1)))   # flops per row
    if name == "tsqr_rhs":
        # split leaf, pass B: Y^T Y and Y^T b' per row (the chunk reflectors' Gram products)
        k1 = k_cols if k1 is None else k1
        return "alu", float(2 * k1 * k1 + 2 * k1 * (k_cols - k1))
    if name == "omega_apply":
        return "alu", 2.0                       # flops per (row x column x rhs) unit
    return None, None


# ------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ------------------------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def oracle_sample(cfg, R):
    """One bounded sample of the oracle's own AZ (O2: oracle/az.py, the paper's Alg. 1 with numpy FFT
    operators, fp64) on this workload, and the full-solve time it implies.

    Timed, every call: the Philox generation and the step-1 operator (A - A Z* A) of 2 of the R probe
    columns; b' = (I - A Z*) b and the step-2 correction Z*(b - A x2) for 2 of the nrhs right-hand
    sides; 2 columns of x2 = Omega y; and the dense SVD of a full-size rows x R sketch.  The solve time
    is ESTIMATED by scaling the per-column parts linearly to R probes / nrhs right-hand sides (every
    column costs the same FFTs) and adding the full-size SVD once.  Returns (estimate_s, sample_s, desc)."""
    from oracle import az as OA
    from oracle import philox as OP
    prob = OA.make_problem(cfg, "fft")
    b = I.rhs(cfg)
    nr = cfg.nrhs
    kc, kr = min(2, R), min(2, nr)
    t_all = time.perf_counter()
    t = time.perf_counter()
    Om = OP.probe_matrix(cfg, list(range(kc)), cfg.seed)
    t_gen = time.perf_counter() - t
    t = time.perf_counter()
    S2 = OA.step1_apply(prob, Om)
    t_probe = time.perf_counter() - t
    t = time.perf_counter()
    OA.resid_apply(prob, b[:, :kr])
    x2 = Om[:, :1] @ np.ones((1, kr))
    prob.apply_Zstar(b[:, :kr] - prob.apply_A(x2))
    t_rhs = time.perf_counter() - t
    rng = np.random.default_rng(0)
    Sfull = rng.standard_normal((S2.shape[0], R))
    t = time.perf_counter()
    np.linalg.svd(Sfull, full_matrices=False)
    t_svd = time.perf_counter() - t
    sample_s = time.perf_counter() - t_all
    est = (R / kc) * (t_gen + t_probe) + (nr / kr) * t_rhs + t_svd + (R / kc) * t_gen
    desc = (f"O2 (oracle/az.py Alg. 1, numpy FFT operators, fp64 -- a CPU AZ) on {cfg.name}: timed {kc} of {R} "
            f"probe columns (Philox + (A - A Z* A)), {kr} of {nr} RHS (b' and step 2), {kc} Omega columns and "
            f"the full-size SVD of a {S2.shape[0]} x {R} sketch ({sample_s:.1f} s); the solve time is ESTIMATED "
            f"by scaling the per-column parts to {R} probes / {nr} RHS")
    return est, sample_s, desc


def o1_timings(max_seconds=25.0):
    """The dense O1 oracle (entrywise A + LAPACK SVD-truncated least squares,
    oracle/az.py tsvd_lsq, multithreaded LAPACK) timed as a whole solve, on c1 and on the largest
    member of the c2 family that fits the time budget; c4's committed golden run is quoted from its
    record (tests/golden/c4_o1.npz, made by tests/golden/make_o1_golden.py)."""
    from oracle import az as OA
    from oracle import dense as OD
    out = {}
    spent = 0.0
    for cfg in (I.get_config("c1"), I.make_config("interval", 1024, nrhs=64, R=64, seed=1),
                I.make_config("interval", 2048, nrhs=64, R=64, seed=1),
                I.make_config("interval", 4096, nrhs=64, R=64, seed=1)):
        t = time.perf_counter()
        A = OD.assemble_A(cfg)
        b = I.rhs(cfg)
        OA.tsvd_lsq(A, b, cfg.tol)
        dt = time.perf_counter() - t
        spent += dt
        out[cfg.name] = {"s_per_solve": dt, "solves_per_s": 1.0 / dt, "rows": int(A.shape[0]), "cols": int(A.shape[1]),
                         "nrhs": cfg.nrhs, "measured": True}
        if spent + 8 * dt > max_seconds:      # the next size costs ~8x (SVD ~ m n^2)
            break
    g = os.path.join(ROOT, "tests", "golden", "c4_o1.npz")
    if os.path.exists(g):
        d = np.load(g)
        out["c4"] = {"s_per_solve": float(d["assemble_s"] + d["svd_s"]), "rows": 19632, "cols": 16384,
                     "measured": "on the build container (tests/golden/c4_o1.npz), not in this run",
                     "threads": int(d["threads"])}
    out["c2"] = {"measured": False, "why": "dense A would be 2^20 x 2^20 (8.8 TB), SURVEY.md §8(c) F5"}
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count()
    if args.warmup > 0:
        oracle_sample(cfg, cfg.R)
    ests, samples = [], []
    desc = ""
    for _ in range(args.steps):
        est, sample_s, desc = oracle_sample(cfg, cfg.R)
        ests.append(est)
        samples.append(sample_s)
    sec = statistics.mean(ests)
    value = 1.0 / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": statistics.mean(samples) * 1e3,
            "ms_per_step_note": "wall time of one bounded oracle sample (what each step actually ran)",
            "estimated_ms_per_solve": sec * 1e3, "extrapolated": True,
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": cfg.n, "L": cfg.s, "nrhs": cfg.nrhs, "R": cfg.R, "tol": cfg.tol},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             "extrapolated": True},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# the other BASELINE configs (c1, c3, c4, c5): fewer timed steps, stated per config
# ------------------------------------------------------------------------------------------
EXTRA_STEPS = {"c1": (3, 50), "c3": (1, 2), "c4": (1, 3), "c5": (1, 1)}   # (warmup, timed steps)


def qr_flops(rows, kp, nrhs):
    """Householder QR of the rows x kp sketch with nrhs columns carried: 2 rows kp^2 - 2/3 kp^3
    (the factorisation) + 4 rows kp nrhs (applying the reflectors to b')."""
    return 2.0 * rows * kp * kp - 2.0 / 3.0 * kp ** 3 + 4.0 * rows * kp * nrhs


def measure_config(name, dev, flush):
    import torch
    from paper_2308_14490_b200 import api, _lib
    cfg = I.get_config(name)
    warm, steps = EXTRA_STEPS[name]
    theta = max(cfg.tol * 1e-2, 1e-12)
    max_blocks = 4 if cfg.dim == 1 else (16 if cfg.n < 512 else 6)
    t0 = time.perf_counter()
    plan = api.Plan.from_config(cfg)
    plan_s = time.perf_counter() - t0
    b = api.colmajor(torch.from_numpy(I.rhs(cfg)).to(dev))
    x = api.empty_colmajor(plan.N, cfg.nrhs, dev)
    ws = torch.empty(plan.solve_workspace_bytes(cfg.nrhs, cfg.R, max_blocks), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warm):
        plan.solve(b, theta, cfg.R, max_blocks, x=x, workspace=ws)
    torch.cuda.synchronize()
    clocks = Clocks(dev.index or 0)
    # the sub-millisecond config (c1) is timed untraced -- its repeated solve replays a CUDA graph, which
    # tracing (two events per launch) disables -- and its kernel breakdown taken from one more, traced
    # solve; the second-long configs are traced inside the timed steps (the events cost microseconds)
    small = name == "c1"
    api.trace_enable(not small)
    ms, reps = [], []
    for i in range(steps):
        flush.fill_(i & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, rep = plan.solve(b, theta, cfg.R, max_blocks, x=x, workspace=ws)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        reps.append(rep)
    if small:
        api.trace_enable(True)
        plan.solve(b, theta, cfg.R, max_blocks, x=x, workspace=ws)
        torch.cuda.synchronize()
    trace = api.trace_report()
    api.trace_enable(False)
    trace_steps = 1 if small else steps
    clk = clocks.stop()
    rep = reps[-1]
    mean = sum(ms) / len(ms)
    qr_ms = sum(v[1] for k, v in trace.items() if k.startswith("qrw_") or k.startswith("tsqr")) / trace_steps
    svd_ms = sum(v[1] for k, v in trace.items() if k.startswith("bjac") or k == "jacobi_svd") / trace_steps
    fl = qr_flops(plan.rows, rep["probes"], cfg.nrhs)
    out = {"solves_per_s": 1000.0 / mean, "ms_per_solve": mean, "steps": steps, "warmup": warm,
           "max_blocks": max_blocks, "plan_s": plan_s, "probes": rep["probes"], "rank": rep["rank"],
           "saturated": rep["saturated"], "probe_applies_per_s": rep["probes"] / (rep["ms_sketch"] * 1e-3)
           if rep["ms_sketch"] else None,
           "stages_ms": {k: rep[k] for k in ("ms_rhs", "ms_sketch", "ms_qr", "ms_svd", "ms_step2")},
           "qr": {"ms": qr_ms, "flops": fl, "tflops": fl / (qr_ms * 1e-3) / 1e12 if qr_ms else None,
                  "frac_fp64": fl / (qr_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS if qr_ms else None},
           "svd_ms": svd_ms,
           "top_kernels_ms": {k: round(v[1] / trace_steps, 3) for k, v in sorted(trace.items(), key=lambda kv: -kv[1][1])[:8]},
           "traced": "timed steps" if not small else "one extra solve after the untraced timed steps",
           "solve_graphs": int(_lib.lib().az_solve_graph_count(plan._h)),
           "clocks": clk}
    del ws, x, b
    plan.close()
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(args, cfg):
    import torch
    from paper_2308_14490_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and not args.replicas:
        # several GPUs: ONE solve sharded over the ranks (az_solve_sharded: the probe / RHS column shards,
        # the NCCL all-to-all re-block and the factor all-gathers; strong scaling).  --replicas times
        # independent single-GPU solves instead (weak scaling, no data-path collective).
        args.sharded = True
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", init_method="env://")
    elif args.sharded:          # the sharded path is collective even on one GPU
        import socket
        import torch.distributed as dist
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    theta = max(cfg.tol * 1e-2, 1e-12)
    max_blocks = 1 if cfg.dim == 1 else 8

    plan = api.Plan.from_config(cfg)
    b_host = I.rhs(cfg)
    b = torch.from_numpy(b_host).to(dev)
    b = api.colmajor(b)
    x = api.empty_colmajor(plan.N, cfg.nrhs, dev)
    ws = torch.empty(plan.solve_workspace_bytes(cfg.nrhs, cfg.R, max_blocks), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > L2 (126 MB)

    if args.sharded:
        # az_solve_sharded: the multi-GPU solve inside libaz (NCCL all-to-all + all-gathers over
        # NVLink, fixed 8-leaf TSQR tree); torch.distributed only bootstraps the communicator
        comm = api.Comm.from_process_group()

        def step(bb=None):
            return api.solve_sharded(plan, comm, b if bb is None else bb, theta, cfg.R, max_blocks, x=x)
    else:
        def step():
            return plan.solve(b, theta, cfg.R, max_blocks, x=x, workspace=ws)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    clocks = Clocks(local)
    api.launch_count(reset=True)
    api.trace_enable(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    reps = []
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)                       # evict L2 between timed iterations (not timed)
        ev[i][0].record(stream)
        _, rep = step()
        ev[i][1].record(stream)
        reps.append(rep)
    torch.cuda.synchronize()
    launches = api.launch_count()
    trace = api.trace_report()
    api.trace_enable(False)
    clk = clocks.stop()
    ms = [a.elapsed_time(bb) for a, bb in ev]
    ms_step = sum(ms) / len(ms)
    if dist:
        t = torch.tensor([ms_step], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())

    # ---- factorisation reuse: factor once, then solve with new RHS ----
    factored = None
    if not args.sharded:
        fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fe0.record(stream)
        fac = api.Factor(plan, theta, cfg.R, max_blocks)
        fe1.record(stream)
        torch.cuda.synchronize()
        fws = torch.empty(fac.workspace_bytes(cfg.nrhs), dtype=torch.uint8, device=dev)
        for _ in range(2):
            fac.solve(b, x=x, workspace=fws)
        torch.cuda.synchronize()
        kf = max(3, min(args.steps, 10))
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(kf)]
        for i in range(kf):
            flush.fill_(i & 0xFF)
            fev[i][0].record(stream)
            fac.solve(b, x=x, workspace=fws)
            fev[i][1].record(stream)
        torch.cuda.synchronize()
        fms = sum(a.elapsed_time(bb) for a, bb in fev) / kf
        api.trace_enable(True)
        fac.solve(b, x=x, workspace=fws)
        ftr = api.trace_report()
        api.trace_enable(False)
        factored = {"solves_per_s": world * 1000.0 / fms, "ms_per_solve": fms, "ms_factorize": fe0.elapsed_time(fe1),
                    "probes": fac.report["probes"], "rank": fac.report["rank"],
                    "kernels_ms": {k: round(v[1], 3) for k, v in sorted(ftr.items(), key=lambda kv: -kv[1][1])[:8]},
                    "note": "az_solve_factored: b' = (I - A Z*) b, c = Q1^T b' (Q1 explicit, formed at factorisation), "
                            "y = P c, x2 = Omega y (Omega stored), step 2"}
        fac.close()
        del fws

    # ---- end to end: every step uploads its b from pinned host memory, solves, and downloads
    # its x to pinned host memory.  Steps are pipelined the way a serving loop would run them:
    # step i+1's upload (copy engine H2D) and step i-1's download (copy engine D2H) overlap
    # step i's solve; the timed region spans the first upload to the last download.
    bh = torch.from_numpy(np.asfortranarray(b_host)).t().contiguous().pin_memory().t()
    xh = [torch.empty((cfg.nrhs, plan.N), dtype=torch.float64).pin_memory().t() for _ in range(2)]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    bdev = [torch.empty_like(b) for _ in range(2)]
    xdev = [api.empty_colmajor(plan.N, cfg.nrhs, dev) for _ in range(2)]

    def e2e_run(k):
        if not args.sharded:
            # the C-ABI host-buffer path: az_solve_host_pipelined (H2D, solve, D2H per step, enqueued;
            # neighbouring steps' copies overlap the solve) + az_plan_sync
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for i in range(k):
                api.solve_host_pipelined(plan, bh, xh[i % 2], theta, cfg.R, max_blocks)
            api.plan_sync(plan)
            t1.record(stream)
            torch.cuda.synchronize()
            return t0.elapsed_time(t1)
        ev_up = [torch.cuda.Event() for _ in range(2)]
        ev_solved = [torch.cuda.Event() for _ in range(2)]
        ev_down = [torch.cuda.Event() for _ in range(2)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(up)
        with torch.cuda.stream(up):
            bdev[0].copy_(bh, non_blocking=True)
            ev_up[0].record(up)
        for i in range(k):
            sl = i % 2
            if i + 1 < k:
                nx = (i + 1) % 2
                with torch.cuda.stream(up):
                    up.wait_event(ev_solved[nx])          # the solve that last read bdev[nx] is done
                    bdev[nx].copy_(bh, non_blocking=True)
                    ev_up[nx].record(up)
            stream.wait_event(ev_up[sl])
            stream.wait_event(ev_down[sl])                # xdev[sl] has been downloaded
            xs, _ = step(bdev[sl])
            xdev[sl].copy_(xs)
            ev_solved[sl].record(stream)
            with torch.cuda.stream(down):
                down.wait_event(ev_solved[sl])
                xh[sl].copy_(xdev[sl], non_blocking=True)
                ev_down[sl].record(down)
        t1.record(down)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    e2e_run(2)
    ke = max(3, args.steps)   # the same K as the device-timed steps (fill and drain amortised alike)
    e2e_ms = e2e_run(ke) / ke
    # the copy engines alone (what e2e can at best overlap the solve with)
    c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    torch.cuda.synchronize()
    c0.record(stream)
    bdev[0].copy_(bh, non_blocking=True)
    c1.record(stream)
    xh[0].copy_(xdev[0], non_blocking=True)
    c2.record(stream)
    torch.cuda.synchronize()
    pcie = {"h2d_gbs": b_host.nbytes / (c0.elapsed_time(c1) * 1e-3) / 1e9,
            "d2h_gbs": plan.N * cfg.nrhs * 8 / (c1.elapsed_time(c2) * 1e-3) / 1e9}
    # both directions at once, as in the pipelined loop: the floor the e2e step time can reach
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    d0.record(stream)
    up.wait_event(d0)
    down.wait_event(d0)
    with torch.cuda.stream(up):
        bdev[0].copy_(bh, non_blocking=True)
    with torch.cuda.stream(down):
        xh[1].copy_(xdev[1], non_blocking=True)
    stream.wait_stream(up)
    stream.wait_stream(down)
    d1.record(stream)
    torch.cuda.synchronize()
    bidir_ms = d0.elapsed_time(d1)
    pcie["bidir_gbs"] = (b_host.nbytes + plan.N * cfg.nrhs * 8) / (bidir_ms * 1e-3) / 1e9
    pcie["bidir_ms_per_step"] = bidir_ms
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (live CUDA-event trace over the timed region) ----
    peaks, peak_src = measured_peaks()
    kcols = reps[-1]["probes"] + cfg.nrhs
    # (a "_bg" pass runs on the lowest-priority stream and yields SMs to the critical branches: its
    # event-timed duration is not its cost, so it is neither the dominant kernel nor in the pass roofline)
    fg = {k: v for k, v in trace.items() if not k.endswith("_bg")}
    dom = max(fg.items(), key=lambda kv: kv[1][1])
    name, (cnt, tot_ms, units) = dom
    # the four-step narrow solve takes Z* b and M = Omega - Z* A Omega from its chains (az_solve.cu step2_linear)
    kept = (cfg.dim == 1 and cfg.N * cfg.s > 2048 and kcols <= 128
            and os.environ.get("AZ_STEP2_LINEAR", "1") != "0")
    split = (kcols <= 128 and reps[-1]["probes"] <= 64 and cfg.nrhs <= 64 and max_blocks == 1
             and not args.sharded and os.environ.get("AZ_TSQR_SPLIT", "1") != "0")
    bound, per_unit = kernel_model(name, cfg, plan.M, kcols, reps[-1]["probes"], kept, split)
    roof = {"kernel": name, "launches": cnt, "ms_total": tot_ms, "share_of_step": tot_ms / sum(ms)}
    if bound == "hbm":
        achieved = per_unit * units / (tot_ms * 1e-3) / 1e9
        roof.update({"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": achieved / peaks["hbm_gbs"], "peak_source": peak_src})
    elif bound == "alu":
        achieved = per_unit * units / (tot_ms * 1e-3) / 1e12
        roof.update({"bound": "alu", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS,
                     "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk x 2 x 1965 MHz (DESIGN.md)"})
    else:
        roof.update({"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None})
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(name)
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    # aggregate HBM roofline of the FFT operator passes (SURVEY.md §8(d) pass model)
    fb, ft = 0.0, 0.0
    for k, (c_, t_, u_) in fg.items():
        bnd, pu = kernel_model(k, cfg, plan.M, kcols, kept=kept)
        if bnd == "hbm":
            fb += pu * u_
            ft += t_
    roof_fft = None
    if ft > 0:
        ach = fb / (ft * 1e-3) / 1e9
        roof_fft = {"kernels": "all FFT operator passes", "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                    "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "share_of_step": ft / sum(ms),
                    "bytes_per_step": fb / args.steps, "peak_source": peak_src,
                    "background_excluded": sorted(k for k in trace if k.endswith("_bg"))}
    # per-kernel table (share of the step)
    kernels = {k: {"launches": v[0], "ms_per_step": v[1] / args.steps, "units": v[2]} for k, v in
               sorted(trace.items(), key=lambda kv: -kv[1][1])}

    rep = reps[-1]
    value = (1 if args.sharded else world) * 1000.0 / ms_step
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        est, sample_s, desc = oracle_sample(cfg, cfg.R)
        cpu = {"value": 1.0 / est, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": desc,
               "extrapolated": True, "sample_s": sample_s, "o1_dense": o1_timings()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong" if args.sharded else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": cfg.name, "n": cfg.n, "L": cfg.s, "dim": cfg.dim, "nrhs": cfg.nrhs, "R": cfg.R,
                   "tol": cfg.tol, "theta": theta, "max_blocks": max_blocks,
                   "parallelism": (f"az_solve_sharded over {world} (NCCL all-to-all re-block, 8-leaf TSQR tree)" if args.sharded
                                   else f"replicas{world}"),
                   "l2": "flushed between timed steps (256 MB write); S alone is 1.07 GB"},
        "probe_applies_per_s": world * rep["probes"] / (rep["ms_sketch"] * 1e-3) if rep["ms_sketch"] else None,
        "rhs_per_s": value * cfg.nrhs,
        "stages_ms": {k: rep[k] for k in ("ms_rhs", "ms_sketch", "ms_qr", "ms_svd", "ms_step2", "ms_total")},
        "rank": rep["rank"], "probes": rep["probes"], "saturated": rep["saturated"],
        "roofline": roof,
        "roofline_fft_passes": roof_fft,
        "factored": factored,
        "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": (1 if args.sharded else world) * 1000.0 / e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(b_host.nbytes),
                "d2h_bytes_per_step": int(plan.N * cfg.nrhs * 8), "ms_per_step": e2e_ms,
                "pcie": pcie,
                "how": "az_solve_host_pipelined per step: H2D of b (pinned) -> az_solve -> D2H of x (pinned); "
                       "neighbouring steps' copies overlap the solve on the two copy engines; az_plan_sync at the end"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and args.extra_configs:
        extra = {}
        del ws
        torch.cuda.empty_cache()
        for nm in [c for c in args.extra_configs.split(",") if c]:
            try:
                extra[nm] = measure_config(nm, dev, flush)
            except Exception as exc:      # report, never hide: a failed config is a visible gap
                extra[nm] = {"error": repr(exc)}
        line["other_configs"] = extra
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extra-configs", default="c1,c3,c4,c5",
                    help="other BASELINE configs timed after the headline (fewer steps, stated); '' = none")
    ap.add_argument("--sharded", action="store_true",
                    help="one solve sharded over the ranks (az_solve_sharded: probe/RHS columns + NCCL all-to-all "
                         "re-block, strong scaling); the default whenever WORLD_SIZE > 1")
    ap.add_argument("--replicas", action="store_true",
                    help="with WORLD_SIZE > 1: independent single-GPU solves per rank (weak scaling) instead")
    args = ap.parse_args()
    cfg = I.get_config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
