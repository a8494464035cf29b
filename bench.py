#!/usr/bin/env python
"""Benchmark: NNCA H2 matvec on B200 at BASELINE.json's headline config.

Workload (BASELINE.json configs[2], the N=1M 3D 1/r case the metric names):
N = 1,048,576 points on the unit sphere (normalised N(0, I3), seed 2), FP64,
Laplace kernel 1/(4 pi r) with K(x, x) = 0, octree with <= 64 points per leaf,
eta = sqrt(2), NNCA tolerance 1e-6, x ~ U(-1, 1).  One setup (tree + NNCA),
then repeated matvecs as in an iterative solver: a bench "step" is one H2
matvec.  Synthetic inputs stand in for the paper's datasets.

Reported: effective N^2/s (value), matvec ms, NNCA setup ms, relative L2
error of the GPU matvec against (a) the CPU oracle's FP64 H2 matvec on the
same input and (b) a direct dense sum on 1000 sampled rows.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Multi-GPU: the H2 matvec does not shard (replicas only): each rank
runs an independent replica, value = aggregate N^2/s over ranks (max-over-ranks
time), scaling "weak".
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "H2 matvec ms & effective N^2/s at N=1M 3D 1/r; NNCA setup ms; rel. L2 err"

CONFIGS = {
    # name: (distribution, N, dim, seed, kernel, kernel kwargs, nu, eps, x-dist, nrhs)
    "c0": ("uniform", 4096, 2, 0, "log", {}, 64, 1e-8, "normal", 1),
    "c1": ("uniform", 262144, 3, 1, "laplace-3d", {}, 64, 1e-8, "normal", 1),
    "c2": ("sphere", 1048576, 3, 2, "laplace-3d", {}, 64, 1e-6, "uniform", 1),
    "c3": ("gmix", 524288, 3, 3, "gaussian", {"sigma": 0.5}, 64, 1e-8, "labels", 1),
    "c4": ("uniform", 4194304, 2, 4, "coulomb-3d", {}, 128, 1e-10, "normal", 16),
}
HEADLINE = "c2"

# ---- roofline models ----
# Nominal FP64 peak of a B200: 148 SMs x 64 DFMA/clk x 2 flop x the max SM clock (1965 MHz) = 37.2 TFLOP/s.
# MEASURED_PEAKS.json has no FP64 entry; the in-run DFMA probe (h2b_fp64_peak, ~34 TFLOP/s) is printed beside it.
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12
HBM_PEAK_GBS_FALLBACK = 6450.6  # MEASURED_PEAKS.json hbm_gbs when present (read at run time)
# Executed FP64 flops per evaluated pair (DFMA = 2, DADD / DMUL = 1; the MUFU seeds and the integer exponent
# rebase are not counted), one RHS:
#   symmetric kernel (interact_sym.cuh), each unordered pair evaluated once and applied both ways:
#     M2L  r^2 = DADD + 3 DFMA (7); K = DMUL + DFMA + DMUL (4, FP32 seed + one quadratic step);
#          row and column accumulations 2 DFMA (4)                                                   -> 15
#     near r^2 = 3 DADD + 3 DFMA (9); K 4; accumulations 4                                          -> 17
#          (the leaf's own block is evaluated in both orders; the other near pairs once)
#   one-directional kernel (interact.cuh; multi-RHS chunks): M2L 13 + 2 per further RHS, near 15 + 2 per RHS
SYM_FLOPS_M2L, SYM_FLOPS_NEAR = 15, 17
DIR_FLOPS_M2L, DIR_FLOPS_NEAR = 13, 15


def hbm_peak_gbs():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return HBM_PEAK_GBS_FALLBACK, "fallback (last measured copy bandwidth on this pool)"


def make_inputs(cfg, n_override=None):
    from paper_2203_14832_b200 import sampling

    dist, n, dim, seed, kname, kkw, nu, eps, xdist, nrhs = cfg
    if n_override:
        n = n_override
    pts = sampling.make_points(dist, n, dim, seed)
    rng = np.random.default_rng(seed + 100)
    if xdist == "uniform":
        w = rng.uniform(-1.0, 1.0, (n, nrhs))
    elif xdist == "labels":
        w = np.where(rng.random((n, nrhs)) < 0.5, -1.0, 1.0)
    else:
        w = rng.standard_normal((n, nrhs))
    return pts, w if nrhs > 1 else w[:, 0]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    """One process per GPU (torchrun env); NCCL on GPUs, gloo otherwise (CPU tests)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local


def max_over_ranks(x, world):
    """Max of a per-rank float over all ranks (the driver's max-over-ranks timing rule)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def aggregate_value(n_points, ms_per_step_max, world):
    """Replicas: every rank multiplies its own copy of the operator; whole-job N^2/s."""
    return world * float(n_points) ** 2 / (ms_per_step_max * 1e-3)


def oracle_pipeline(pts, cfg, w, threads=None, matvecs=1):
    """The CPU oracle (reference algorithm restated in C, OpenMP): setup + matvecs."""
    from oracle import oracle as O

    if threads:
        O.set_threads(threads)
    kname, kkw, nu, eps = cfg[4], cfg[5], cfg[6], cfg[7]
    kind = {"laplace-3d": 5, "coulomb-3d": 2, "log": 6, "gaussian": 7 if kkw else 4}[kname]
    a = 1.0 / (2.0 * kkw["sigma"] ** 2) if kkw else 0.0
    t0 = time.perf_counter()
    t = O.OTree(pts, None, nu=nu)
    h = O.OH2(t, kind, a, eps)
    setup_s = time.perf_counter() - t0
    times, u = [], None
    for _ in range(matvecs):
        t1 = time.perf_counter()
        u = h.matvec(w)
        times.append(time.perf_counter() - t1)
    return {"setup_s": setup_s, "matvec_s": times, "u": u, "threads": O.threads(), "tree": t, "h2": h}


def run_reference(args, cfg, world, rank):
    """--impl reference: the reference algorithm (CPU oracle) on the host cores."""
    if rank != 0:
        return
    pts, w = make_inputs(cfg, args.n)
    n = pts.shape[0]
    res = oracle_pipeline(pts, cfg, w, matvecs=args.warmup + args.steps)
    times = res["matvec_s"][args.warmup:]
    ms = 1e3 * float(np.mean(times))
    value = n * n / (ms * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "N^2/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, cfg, n),
        "matvec_ms": ms, "setup_ms": 1e3 * res["setup_s"],
        "cpu_baseline": {"value": value, "unit": "N^2/s", "cores": res["threads"], "kind": "port",
                         "sample": f"full workload: oracle setup once + {args.warmup}+{args.steps} full matvecs at "
                                   f"N={n}"},
        "e2e": {"value": value, "unit": "N^2/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args, cfg, n):
    """The workload identity, identical in both arms (the driver compares them)."""
    nrhs = cfg[9]
    return {"workload": workload_name(args, cfg, n), "N": n, "nrhs": nrhs}


def workload_name(args, cfg, n, name=None):
    dist, _, dim, seed, kname, kkw, nu, eps, xdist, nrhs = cfg
    return (f"{name or args.config}: {dist} N={n} d={dim} seed={seed} kernel={kname}{kkw or ''} nu={nu} eps={eps:g} "
            f"x~{xdist} nrhs={nrhs}")


def run_b200(args, cfg, world, rank, local):
    # the engine's stream-ordered pool is reserved up front (common.cuh pool_init); the benchmark owns the
    # GPU, so it reserves enough for the largest configuration's setup (pool growth mid-setup is slow)
    os.environ.setdefault("H2B_POOL_RESERVE_GB", "32")
    import torch

    import paper_2203_14832_b200 as h2c
    from paper_2203_14832_b200 import _lib
    from paper_2203_14832_b200.matvec import matvec_launches, stage_times

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    pts, w = make_inputs(cfg, args.n)
    n = pts.shape[0]
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    kname, kkw, nu, eps = cfg[4], cfg[5], cfg[6], cfg[7]
    kern = h2c.builtin_kernel(kname, cfg[2], **kkw)
    cloud = h2c.PointCloud.from_points(pts)

    # ---- warm-up of the engine on a small problem (lazy CUDA module loading, allocator) ----
    wcloud = h2c.PointCloud.from_points(pts[:: max(1, n // 4096)][:4096])
    h2c.h2_matvec(h2c.assemble(h2c.build_tree(wcloud, nu=nu, eta=float(np.sqrt(2.0))), kern, eps),
                  np.ones(wcloud.n_sources))
    # ---- setup: tree + NNCA (timed on the host around synchronous calls).  Run twice: the first full-size
    # setup also grows the stream-ordered memory pool and loads the large-cell kernel variants the small
    # warm-up did not touch (reported as setup_first_ms); the second is the steady state (setup_ms). ----
    setups = []
    for _ in range(2):
        h2 = tree = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree = h2c.build_tree(cloud, nu=nu, eta=float(np.sqrt(2.0)))
        t1 = time.perf_counter()
        h2 = h2c.assemble(tree, kern, eps)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        setups.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
    tree_ms, nnca_ms = setups[-1]

    stream = torch.cuda.current_stream(dev)
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    ud = torch.empty((n,) if nrhs == 1 else (n, nrhs), dtype=torch.float64, device=dev)
    L = _lib.lib()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def matvec_dev():
        _lib.check(L.h2b_matvec(h2.handle, wd.data_ptr(), ud.data_ptr(), nrhs, 1, stream.cuda_stream))

    for _ in range(args.warmup):
        matvec_dev()
    torch.cuda.synchronize()

    # ---- timed region: K device-resident matvecs, L2 flushed between them ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for e0, e1 in evs:
            flush.zero_()
            e0.record(stream)
            matvec_dev()
            e1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    per = [e0.elapsed_time(e1) for e0, e1 in evs]
    ms = max_over_ranks(float(np.mean(per)), world)
    value = aggregate_value(n, ms, world)

    # ---- e2e: the public drop-in call h2_matvec(h2, w) on pinned host tensors (H2D + matvec + D2H per step,
    # inside the timed region; the call returns after the result is on the host) ----
    wh = torch.from_numpy(np.ascontiguousarray(w)).pin_memory()
    uh = torch.empty(tuple(ud.shape), dtype=torch.float64).pin_memory()
    for _ in range(2):
        h2c.h2_matvec(h2, wh, out=uh)
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier(world)
    for e0, e1 in ee:
        flush.zero_()
        e0.record(stream)
        h2c.h2_matvec(h2, wh, out=uh)
        e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(float(np.mean([e0.elapsed_time(e1) for e0, e1 in ee])), world)
    e2e_value = aggregate_value(n, e2e_ms, world)
    # the same call on numpy arrays, host wall clock (reported beside, not the headline): ordinary pageable
    # arrays (the driver stages the copies), and arrays from h2c.pinned_empty (page-locked: same path as above)
    def wall_ms(wv, uv):
        h2c.h2_matvec(h2, wv, out=uv)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            h2c.h2_matvec(h2, wv, out=uv)
        return 1e3 * (time.perf_counter() - t0) / args.steps

    e2e_numpy_ms = wall_ms(np.ascontiguousarray(w), np.empty(tuple(ud.shape)))
    wp, up = h2c.pinned_empty(w.shape), h2c.pinned_empty(tuple(ud.shape))
    wp[...] = w
    e2e_numpy_pinned_ms = wall_ms(wp, up)

    # ---- roofline of the dominant kernel (FP64 interaction: M2L + near field), the transfer passes and setup ----
    st = h2.native_stats()
    pairs_m2l, pairs_p2p = int(st[1]), int(st[2])
    depth = int(st[8])
    stage = stage_times(h2, wd, repeats=max(3, min(args.steps, 10)))  # [up, m2l+near, l2l, l2p, total]
    probe = ctypes_peak(L)
    sym = bool(st[6]) and nrhs % 16 != 0
    leaf_sizes = np.diff(tree.array(depth, "t_ptr")) if depth >= 0 else np.zeros(0)
    self_pairs = int(np.sum(leaf_sizes.astype(np.int64) ** 2))
    if sym:
        evaluated = {"m2l": pairs_m2l // 2, "near": (pairs_p2p - self_pairs) // 2 + self_pairs}
        flops = evaluated["m2l"] * SYM_FLOPS_M2L + evaluated["near"] * SYM_FLOPS_NEAR
        fpp = {"m2l": SYM_FLOPS_M2L, "near": SYM_FLOPS_NEAR, "per": "evaluated unordered pair"}
    else:
        evaluated = {"m2l": pairs_m2l, "near": pairs_p2p}
        flops = pairs_m2l * (DIR_FLOPS_M2L + 2 * (nrhs - 1)) + pairs_p2p * (DIR_FLOPS_NEAR + 2 * (nrhs - 1))
        fpp = {"m2l": DIR_FLOPS_M2L + 2 * (nrhs - 1), "near": DIR_FLOPS_NEAR + 2 * (nrhs - 1),
               "per": "applied entry (one-directional kernel)"}
    inter_ms = stage[1]
    achieved = flops / (inter_ms * 1e-3) / 1e12
    traffic, traffic_src = load_traffic(args.config)
    hbm_peak, hbm_src = hbm_peak_gbs()
    # transfer passes: algorithmic bytes = the interpolation operators read once per product (P2M / M2M read
    # the column interpolators, L2L / L2P the row interpolators; pmat per level = sum over cells of rows x k) plus
    # the coefficient vectors they stream (w in, pivot coefficients written and read, u out), nrhs columns each
    op_bytes = dense_op_bytes = idx_bytes = 0
    vec_bytes = 8 * nrhs * (2 * n)  # w_sorted read + u written (near-field partials read by L2P: + n)
    vec_bytes += 8 * nrhs * n
    for lev in range(2, depth + 1):
        m_in, k_in = h2.array(lev, "m_in"), h2.array(lev, "k_in")
        n_out, k_out = h2.array(lev, "n_out"), h2.array(lev, "k_out")
        # compact operators (csrc/transfer.cuh): the k identity rows of every interpolator are not stored
        op_bytes += 8 * int(np.dot(m_in - k_in, k_in)) + 8 * int(np.dot(n_out - k_out, k_out))
        dense_op_bytes += 8 * int(np.dot(m_in, k_in)) + 8 * int(np.dot(n_out, k_out))
        # row maps: position (+ owner downward) per general row, identity-row position (+ owner upward) per pivot
        idx_bytes += 4 * (int((n_out - k_out).sum()) + 2 * int(k_out.sum()))
        idx_bytes += 4 * (2 * int((m_in - k_in).sum()) + int(k_in.sum()))
        vec_bytes += 8 * nrhs * 4 * int(k_in.sum())  # coefficients: written + read up, read + written down
    tr_ms = stage[0] + stage[2] + stage[3]
    tr_bytes = op_bytes + idx_bytes + vec_bytes
    # setup: the ACA's residual sweeps (reference operation order, _core.pyx:70-191): step t re-reads the t previous
    # residual rows / columns of the cell's block (n + m entries each), once for the residual and once for the
    # stopping test's cross products.  nevals per cell ~ k (n + m), so operand bytes ~ 8 (k - 1) nevals and
    # FP64 flops ~ 4 (k - 1) / 2 * 2 nevals (one FMA per operand entry and sweep)
    aca_bytes = aca_flops = 0
    for lev in range(2, depth + 1):
        k_in, nev = h2.array(lev, "k_in").astype(np.float64), h2.array(lev, "nevals").astype(np.float64)
        aca_bytes += 8.0 * float(np.dot(np.maximum(k_in - 1, 0), nev))
        aca_flops += 2.0 * float(np.dot(np.maximum(k_in - 1, 0), nev))
    setup_s = (tree_ms + nnca_ms) * 1e-3
    roof_inter = {"bound": "fp64", "kernel": "interact_sym (M2L all levels + near field)" if sym else
                  "interact_warps (M2L all levels + near field)",
                  "achieved": achieved, "peak": NOMINAL_FP64_TFLOPS, "unit": "TFLOP/s",
                  "frac": achieved / NOMINAL_FP64_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                  "peak_source": "nominal B200 FP64 (148 SM x 64 DFMA/clk x 2 x 1965 MHz); MEASURED_PEAKS.json "
                                 "has no FP64 entry",
                  "fp64_probe_tflops": probe, "frac_of_probe": achieved / probe,
                  "flops": flops, "ms": inter_ms, "flops_per_pair": fpp, "evaluated_pairs": evaluated,
                  "applied_entries_per_s": (pairs_m2l + pairs_p2p) / (inter_ms * 1e-3),
                  # the same launch measured in the units of DESIGN.md (applied entries) at the flops an entry costs
                  # when every ordered pair is evaluated (13 / 15 per entry, what the one-directional kernel
                  # executes): the symmetric kernel applies each evaluated pair twice, so this exceeds `achieved`
                  "effective": {"flops_per_applied_entry": {"m2l": DIR_FLOPS_M2L, "near": DIR_FLOPS_NEAR},
                                "achieved": (pairs_m2l * DIR_FLOPS_M2L + pairs_p2p * DIR_FLOPS_NEAR) /
                                            (inter_ms * 1e-3) / 1e12,
                                "frac": (pairs_m2l * DIR_FLOPS_M2L + pairs_p2p * DIR_FLOPS_NEAR) /
                                        (inter_ms * 1e-3) / 1e12 / NOMINAL_FP64_TFLOPS} if nrhs == 1 else None}
    roof_tr = {"bound": "hbm", "kernel": "up_compact/down_compact (P2M, M2M, L2L, L2P on compact interpolators)",
               "achieved": tr_bytes / (tr_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
               "frac": tr_bytes / (tr_ms * 1e-3) / 1e9 / hbm_peak, "bytes": tr_bytes, "operator_bytes": op_bytes,
               "dense_operator_bytes": dense_op_bytes,
               "ms": tr_ms, "peak_source": hbm_src}
    roof_setup = {"n2_per_s": float(n) ** 2 / setup_s, "ms": setup_s * 1e3,
                  "aca_operand_bytes_model": aca_bytes, "aca_achieved_GBps": aca_bytes / (nnca_ms * 1e-3) / 1e9,
                  "aca_frac_hbm": aca_bytes / (nnca_ms * 1e-3) / 1e9 / hbm_peak,
                  "aca_flops_model": aca_flops, "aca_achieved_tflops": aca_flops / (nnca_ms * 1e-3) / 1e12,
                  "aca_frac_fp64": aca_flops / (nnca_ms * 1e-3) / 1e12 / NOMINAL_FP64_TFLOPS,
                  "note": "model bytes / flops of the residual sweeps.  ncu (profiles/r2j_aca_ring_ncu_full.json): the ACA "
                          "kernel is issue / latency bound at the leaves (issue slots 35% busy at 16 warps per SM, FP64 pipe 13%) and "
                          "DRAM-bound on the residual rows at the levels above (5.3 TB/s at level 6)"}

    # ---- accuracy: sampled dense rows + CPU-oracle H2 matvec at the full N ----
    uhost = ud.cpu().numpy()
    rng = np.random.default_rng(7)
    rows = rng.choice(n, size=min(1000, n), replace=False)
    wcol = w if nrhs == 1 else w[:, 0]
    exact = h2c.dense_rows(kern, cloud, rows, wcol)
    ucol = uhost if nrhs == 1 else uhost[:, 0]
    err_dense = float(np.linalg.norm(ucol[rows] - exact) / np.linalg.norm(exact))

    line = {
        "metric": METRIC, "value": value, "unit": "N^2/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; stands in for the paper's point sets)",
        "config": config_dict(args, cfg, n),
        "l2": "flushed (256 MB write) between timed steps", "parallelism": f"replicas x{world}",
        "matvec_ms": ms, "setup_ms": tree_ms + nnca_ms, "tree_ms": tree_ms, "nnca_ms": nnca_ms,
        "setup_first_ms": sum(setups[0]), "setup_n2_per_s": float(n) ** 2 / setup_s,
        "depth": depth, "max_rank": int(st[3]), "m2l_pairs": pairs_m2l, "p2p_pairs": pairs_p2p,
        "stage_ms": {"upward": stage[0], "interaction": stage[1], "l2l": stage[2], "l2p": stage[3],
                     "total": stage[4]},
        "rel_l2_err_dense_1000_rows": err_dense, "eps": cfg[7], "eps_ratio": err_dense / cfg[7],
        "e2e": {"value": e2e_value, "unit": "N^2/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": int(wh.nbytes),
                "d2h_bytes_per_step": int(uh.nbytes),
                "call": "paper_2203_14832_b200.h2_matvec(h2, w_pinned, out=u_pinned) (C ABI h2b_matvec, host "
                        "pointers)"},
        "e2e_numpy_ms": e2e_numpy_ms, "e2e_numpy_pinned_ms": e2e_numpy_pinned_ms,
        # the north star's use case at this config: one setup, then 50 products (iterative solver), end to end
        "solver_use_case_ms": {"setup": tree_ms + nnca_ms, "50_matvecs_e2e": 50 * e2e_ms,
                               "total": tree_ms + nnca_ms + 50 * e2e_ms},
        "gpu_launches": int(matvec_launches(h2, nrhs)) * args.steps,
        "roofline": dict(roof_inter, transfers=roof_tr, setup=roof_setup),
        "clocks": clk.summary(),
    }
    if rank == 0 and args.config == HEADLINE and not args.no_other_configs and args.n is None and world == 1:
        # the other BASELINE configs at their stated sizes (parity for them: tests/test_baseline_configs.py)
        h2 = tree = None
        del wd, ud, flush
        torch.cuda.empty_cache()
        line["other_configs"] = {name: side_config(args, name, dev) for name in ("c0", "c1", "c3", "c4")}
    if rank == 0 and not args.no_cpu_baseline and args.gpus == 1 and world == 1:
        res = oracle_pipeline(pts, cfg, w, matvecs=1)
        cpu_ms = 1e3 * res["matvec_s"][0]
        uo = res["u"]
        line["rel_l2_err_vs_oracle_h2"] = float(np.linalg.norm(uhost - uo) / np.linalg.norm(uo))
        line["cpu_baseline"] = {"value": n * n / (cpu_ms * 1e-3), "unit": "N^2/s", "cores": res["threads"],
                                "kind": "port", "matvec_ms": cpu_ms, "setup_ms": 1e3 * res["setup_s"],
                                "sample": f"full workload once: oracle tree+NNCA setup and one full H2 matvec at "
                                          f"N={n} (OpenMP, all host threads)"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def side_config(args, name, dev):
    """Setup and device-resident product of another BASELINE config (same timing rules, 5 timed products)."""
    import torch

    import paper_2203_14832_b200 as h2c

    cfg = CONFIGS[name]
    pts, w = make_inputs(cfg)
    n = pts.shape[0]
    nrhs = 1 if w.ndim == 1 else w.shape[1]
    kern = h2c.builtin_kernel(cfg[4], cfg[2], **cfg[5])
    cloud = h2c.PointCloud.from_points(pts)
    setups = []
    for _ in range(2):
        h2 = tree = None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tree = h2c.build_tree(cloud, nu=cfg[6], eta=float(np.sqrt(2.0)))
        t1 = time.perf_counter()
        h2 = h2c.assemble(tree, kern, cfg[7])
        torch.cuda.synchronize()
        setups.append((1e3 * (t1 - t0), 1e3 * (time.perf_counter() - t1)))
    wd = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    ud = torch.empty_like(wd)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        h2c.h2_matvec(h2, wd, out=ud)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        h2c.h2_matvec(h2, wd, out=ud)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in evs]))
    rows = np.random.default_rng(7).choice(n, size=min(1000, n), replace=False)
    wcol = w if nrhs == 1 else np.ascontiguousarray(w[:, 0])
    exact = h2c.dense_rows(kern, cloud, rows, wcol)
    u = ud.cpu().numpy()
    ucol = u if nrhs == 1 else u[:, 0]
    err = float(np.linalg.norm(ucol[rows] - exact) / np.linalg.norm(exact))
    st = h2.native_stats()
    out = {"workload": workload_name(args, cfg, n, name), "N": n, "nrhs": nrhs, "matvec_ms": ms,
           "n2_per_s": nrhs * float(n) ** 2 / (ms * 1e-3), "tree_ms": setups[-1][0], "nnca_ms": setups[-1][1],
           "setup_first_ms": sum(setups[0]), "depth": int(st[8]), "max_rank": int(st[3]),
           "rel_l2_err_dense_1000_rows": err, "eps": cfg[7], "eps_ratio": err / cfg[7]}
    h2 = tree = None
    h2c.release_workspace()  # the next config sizes its own ACA arena
    return out


def ctypes_peak(L):
    import ctypes

    v = ctypes.c_double()
    L.h2b_fp64_peak(ctypes.byref(v))
    return v.value


def load_traffic(config):
    """DRAM bytes per launch of the interaction kernel (dram__bytes_read.sum + dram__bytes_write.sum) from the
    committed ncu --set full capture of the current kernel, if any (profiles/interact_traffic.json)."""
    path = os.path.join(REPO, "profiles", "interact_traffic.json")
    try:
        d = json.load(open(path))
        e = d.get(config)
        if e:
            return e["dram_bytes_per_launch"], e["source"]
    except (OSError, ValueError, KeyError):
        pass
    return None, "no ncu capture of this kernel at this config committed"


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--n", type=int, default=None, help="override N (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the setup + product timings of the other BASELINE configs (c0, c1, c3, c4)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
    else:
        run_b200(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
