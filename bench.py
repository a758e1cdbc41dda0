#!/usr/bin/env python3
"""Benchmark of the B200 T / T* / CGLS hot path (BASELINE.json metric:
"T.x+T*.y pairs/sec and CGLS iters/sec; % of HBM/FP64 roofline at 1/2/4/8 GPU").

Default workload = C5 (BASELINE.json configs[4]): 256 independent 2D
non-uniform problems, each 2^18 jittered-grid samples (spacing 0.5 on
[-128,128)^2, U(-0.2,0.2) jitter, seed 20160613+b), db4 at J=8 (256x256
coefficients), Voronoi density weights, complex128 coefficients and noise
sigma=1e-3.  It is the configuration the metric's 1/2/4/8-GPU scaling is
quoted on and the largest that fits one GPU.  Problems shard across ranks
(no data-path collective; total work fixed -> "strong" scaling).

A step = one CGLS iteration (solver.cpp:70-88: one T, one T*, the norms and
axpys) over every problem of the rank.  `value` = problem-iterations/s over
all ranks, device-timed with CUDA events (max over ranks).  Inputs (per-point
factor tables, 35 GB at N=1) exceed L2, so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1..c5]
  python bench.py --impl reference ...   # CPU restatement of the reference
                                          # on the host cores (oracle/)
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20160613
WORKLOADS = {
    # name: (dim, family p, J, builder, iterations in the config, noise sigma, description)
    "c1": "1D uniform: M=1024 integer frequencies -512..511, Haar J=9 (N=512), sigma=1e-3",
    "c2": "1D jittered: M=4096 (spacing 0.5, U(-0.2,0.2)), Voronoi weights, db4 J=10 (N=1024), sigma=1e-3",
    "c3": "2D uniform tensor: 512x512 integer grid on [-256,256)^2, db2 J=8 (N=256^2), sigma=1e-4",
    "c4": "2D spiral: 2^20 samples, R=512, 64 turns, Voronoi weights, db4 J=9 (N=512^2), sigma=1e-4",
    "c5": "Batched 2D jittered: 256 problems x 2^18 samples (spacing 0.5 on [-128,128)^2, U(-0.2,0.2)), "
          "Voronoi weights, db4 J=8 (N=256^2), sigma=1e-3",
}


# ------------------------------------------------------------------ inputs
def problem_inputs(workload, b, gen):
    """(dim, p, J, coords, weights, bandwidth, sigma) of problem b, via a generator
    module exposing gen_grid / gen_jitter / gen_spiral / voronoi."""
    if workload == "c1":
        return 1, 1, 9, gen.gen_grid(1024, 1.0), None, 512.0, 1e-3
    if workload == "c2":
        c = gen.gen_jitter(4096, 0.5, 0.2, SEED + b)
        K = float(np.max(np.abs(c)))
        return 1, 4, 10, c, gen.voronoi(1, c, K), K, 1e-3
    if workload == "c3":
        return 2, 2, 8, gen.gen_grid(512, 1.0, 2), None, 256.0, 1e-4
    if workload == "c4":
        c = gen.gen_spiral(64, 16384.0, 512.0)
        return 2, 4, 9, c, gen.voronoi(2, c, 512.0), 512.0, 1e-4
    if workload == "c5":
        c = gen.gen_jitter(512, 0.5, 0.2, SEED + b, 2)
        K = float(np.max(np.abs(c)))
        return 2, 4, 8, c, gen.voronoi(2, c, K), K, 1e-3
    raise SystemExit(f"unknown workload {workload}")


def problem_count(workload):
    return 256 if workload == "c5" else 1


# (dim, family p, J, samples per problem, coefficients per problem, the reference's route)
SHAPES = {"c1": (1, 1, 9, 1024, 512, "uniform_1d"), "c2": (1, 4, 10, 4096, 1024, "nfft_1d"),
          "c3": (2, 2, 8, 262144, 65536, "nfft_2d"), "c4": (2, 4, 9, 1048576, 262144, "nfft_2d"),
          "c5": (2, 4, 8, 262144, 65536, "nfft_2d")}


def config_for(workload, P, world):
    """The `config` object both arms print (identical dicts for the same run)."""
    dim, p, J, M, Nc, route = SHAPES[workload]
    return {"workload": workload.upper(), "description": WORKLOADS[workload], "problems": P,
            "samples_per_problem": M, "coeffs_per_problem": Nc, "family": f"p={p}", "J": J,
            "reference_route": route, "iterations_in_config": CONFIG_ITERS[workload],
            "cgls_tolerance": "1e-300 (fixed count)",
            "parallelism": f"problem-sharded x{world}" if world > 1 else "1 rank"}


def host_cpu():
    """CPU model and physical core count of this host."""
    model, cores = "unknown", set()
    try:
        phys = core = None
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name":
                model = v
            elif k == "physical id":
                phys = v
            elif k == "core id":
                core = v
            elif not k and phys is not None:
                cores.add((phys, core))
                phys = core = None
        if phys is not None:
            cores.add((phys, core))
    except OSError:
        pass
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    return {"model": model, "physical_cores": len(cores) or None, "logical_cpus_available": ncpu}


def coeffs_and_noise(b, ncols, nrows, sigma):
    rng = np.random.default_rng(SEED + 7919 * b)
    x = (rng.standard_normal(ncols) + 1j * rng.standard_normal(ncols)) / math.sqrt(2.0)
    noise = sigma * (rng.standard_normal(nrows) + 1j * rng.standard_normal(nrows)) / math.sqrt(2.0)
    return x, noise


class ProductGen:
    """Input harness of the product package (csrc/host_inputs.cpp)."""

    def __init__(self):
        from paper_1607_04091_b200 import inputs
        self.i = inputs

    def gen_grid(self, M, eps, dim=1):
        return self.i.gen_grid(M, eps, dim)

    def gen_jitter(self, M, eps, eta, seed, dim=1):
        return self.i.gen_jitter(M, eps, eta, seed, dim)

    def gen_spiral(self, t, ppt, K):
        return self.i.gen_spiral(t, ppt, K)

    def voronoi(self, dim, c, K):
        return self.i.voronoi_weights(dim, c, K)  # host threads (GPU cells are bit-identical: test_gpu_voronoi)


# ------------------------------------------------------------------ roofline bookkeeping
E2E_CALLS = 3
# CGLS iterations each config specifies (BASELINE.json configs): one e2e call = one such solve
CONFIG_ITERS = {"c1": 50, "c2": 100, "c3": 100, "c4": 200, "c5": 100}


def algorithmic_bytes(kernel, dim, p, M, Nc, uaxis=None):
    """Compulsory HBM bytes of one launch per problem (SURVEY 8(d) accounting:
    coordinates 8*dim, D 16*dim, L/R 32*p*dim per sample; x / y 16 B per entry).
    Tensor-route passes (`k_uni_*[x-pass|y-pass]`, C3): the pass's input and
    output vectors plus its per-axis factor records (uaxis samples per axis)."""
    per_pt = 8 * dim + 16 * dim + (32 * p * dim if p >= 2 else 0)
    base, tag = kernel.split("[")[0], kernel[len(kernel.split("[")[0]):]
    if base in ("k2_interp", "k2f_interp", "k_n1_interp"):
        return M * (per_pt + 16) + 16 * Nc
    if base in ("k2_spread", "k2f_spread", "k_n1_spread"):
        return M * (per_pt + 16)
    if base in ("k_uni_fwd", "k_uni_adj") and tag and uaxis:
        n = int(round(Nc ** 0.5))
        rec = uaxis * (1 + (2 * p if p >= 2 else 0)) * 16
        mid = 16 * uaxis * n  # the pass-to-pass intermediate W (uaxis x n)
        return (16 * Nc if "x-pass" in tag else 16 * M) + mid + rec
    if base in ("k_uni_fwd", "k_uni_adj"):  # whole 1D uniform apply in one CTA
        return 16 * (Nc + M) + M * (16 + (32 * p if p >= 2 else 0))
    return None


def iteration_bytes(dim, p, M, Nc, uniform_axis=None):
    """bytes per CGLS iteration = pair + 16 (6 Nc + 3 M)."""
    if uniform_axis is not None:
        pair = 2 * (16 * Nc + 16 * M) + 2 * 16 * dim * uniform_axis * (1 + (2 * p if p >= 2 else 0))
    else:
        pair = 2 * (16 * Nc + 16 * M + 8 * dim * M + 16 * dim * M + (32 * p * dim * M if p >= 2 else 0))
    return pair, pair + 16 * (6 * Nc + 3 * M)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def algorithmic_flops(kernel, p, M, S=13, Nc=None):
    """FP64 flops of one launch per problem.  2D gridding: 4 real
    flops per (complex value x real weight) tap over the S x S region and the
    4p side lines of S taps, plus the p x p corner blocks (32 p^2 per sample).
    Direct NDFT (a14): 8 real flops per complex multiply-add term, M x Nc terms."""
    base = kernel.split("[")[0]
    if base in ("k_ndft_fwd", "k_ndft_adj") and Nc:
        return 8 * M * Nc
    if base not in ("k2f_interp", "k2f_spread", "k2_interp", "k2_spread"):
        return None
    return 4 * (S * S + (4 * p * S if p >= 2 else 0)) * M + (32 * p * p * M if p >= 2 else 0)


def load_fp64_peak():
    """FP64 tensor-pipe peak measured on this GPU model (tools/micro/fp64_mix_probe.cu,
    DMMA alone; profiles/fp64_peak.json), else the B200 datasheet FP64 figure."""
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as f:
            d = json.load(f)
        return float(d["dmma_tflops"]), "measured: " + d.get("source", "profiles/fp64_peak.json")
    except Exception:
        return 37.0, "fallback: B200 datasheet FP64"


def load_traffic(kernel, workload):
    """dram bytes per launch per problem from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"gs_clocks_{os.getpid()}_{device}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ distributed plumbing
def dist_init(n):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(v, world, device):
    if world <= 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ GPU arm
def run_gpu(args):
    import torch
    import paper_1607_04091_b200 as gs

    rank, world, local = dist_init(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    gen = ProductGen()
    P = args.problems or problem_count(args.workload)
    lo, hi = rank * P // world, (rank + 1) * P // world
    mine = list(range(lo, hi))
    B = len(mine)
    t0 = time.time()
    inp = [problem_inputs(args.workload, b, gen) for b in mine]
    dim, p, J = inp[0][0], inp[0][1], inp[0][2]
    sigma_noise = inp[0][6]
    bw = max(x[5] for x in inp)
    sets = [gs.SamplingSet(dim, x[3]) for x in inp]
    weighted = inp[0][4] is not None
    mu = np.concatenate([x[4] for x in inp]) if weighted else None
    # data w = T_unweighted x_true + noise; the unweighted operator
    # is built, applied and released before the weighted one is built
    route_kw = dict(allow_tensor_route=args.tensor_route, exact_ndft=args.exact_ndft)
    op_u = gs.freq2wave(sets, p, J, bandwidth=bw, device=local, **route_kw)
    M, Nc = op_u.rows(), op_u.cols()
    xs, ns = zip(*[coeffs_and_noise(b, Nc, M, sigma_noise) for b in mine])
    x_true = torch.from_numpy(np.concatenate(xs)).to(dev)
    data = gs.apply_forward(op_u, x_true) + torch.from_numpy(np.concatenate(ns)).to(dev)
    op_u.close()
    del op_u
    torch.cuda.synchronize()
    op = gs.freq2wave(sets, p, J, bandwidth=bw, weights=mu, device=local, **route_kw)
    route = op.route
    build_s = time.time() - t0
    stream = torch.cuda.current_stream(dev)
    L = gs.load_library()
    import ctypes as C
    L.gs_launch_count.restype = C.c_longlong

    # -------- value: device-timed CGLS iterations over the resident batch
    sess = gs.CglsSession(op, data, tolerance=1e-300, history_capacity=args.warmup + args.steps + 2, stream=stream)
    sess.step(args.warmup, stream=stream)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    n0 = L.gs_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sess.step(args.steps, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = L.gs_launch_count() - n0
    clk = clocks.stop()
    ms = allreduce_max(e0.elapsed_time(e1), world, dev)
    _, st = sess.result()
    sess.close()
    ms_per_step = ms / args.steps
    value = P * args.steps / (ms / 1e3)

    # -------- pairs/s through the public API on resident device tensors
    xp = torch.randn(B * Nc, dtype=torch.complex128, device=dev)
    yp = torch.randn(B * M, dtype=torch.complex128, device=dev)
    for _ in range(2):
        gs.apply_adjoint(op, gs.apply_forward(op, xp, stream=stream), stream=stream)
    torch.cuda.synchronize()
    npairs = max(2, min(args.steps, 10))
    e0.record(stream)
    for _ in range(npairs):
        gs.apply_forward(op, xp, stream=stream)
        gs.apply_adjoint(op, yp, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    pair_ms = allreduce_max(e0.elapsed_time(e1), world, dev) / npairs
    pairs_per_sec = P / (pair_ms / 1e3)

    # -------- per-kernel device times of one pair -> dominant kernel roofline
    prof = gs_profile(op, stream)
    peak, peak_kind = load_peaks()
    uaxis = {"c1": 1024, "c3": 512}.get(args.workload)
    dom = max((k for k in prof if algorithmic_bytes(k, dim, p, M, Nc, uaxis) is not None), key=lambda k: prof[k],
              default=None)
    roofline = None
    fpeak, fpeak_src = load_fp64_peak()
    nd = [k for k in prof if k.startswith("k_ndft_fwd") or k.startswith("k_ndft_adj")]
    if nd and (dom is None or max(prof[k] for k in nd) > prof[dom]):
        # exact NDFT route: the dominant kernel is bound by the FP64 pipe, not HBM
        dom = max(nd, key=lambda k: prof[k])
        fl = algorithmic_flops(dom, p, M, Nc=Nc) * B
        tf = fl / (prof[dom] / 1e3) / 1e12
        roofline = {"bound": "fp64", "kernel": dom, "achieved": round(tf, 3), "peak": fpeak, "unit": "TFLOP/s",
                    "frac": round(tf / fpeak, 4), "traffic": None, "algorithmic_flops_per_launch": fl,
                    "launch_ms": round(prof[dom], 4), "peak_source": fpeak_src}
        dom = None
    if dom is not None:
        ab = algorithmic_bytes(dom, dim, p, M, Nc, uaxis) * B
        ach = ab / (prof[dom] / 1e3) / 1e9
        tr = load_traffic(dom, args.workload)
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 2), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": (tr * B if tr is not None else None),
                    "algorithmic_bytes_per_launch": ab, "launch_ms": round(prof[dom], 4),
                    "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    # FP64 co-limit of the 2D gridding kernels (they issue DMMAs): algorithmic
    # flops per launch / the same live launch time, against the FP64 pipe peak
    roofline_fp64 = {}
    for k in prof:
        fl = algorithmic_flops(k, p, M, Nc=Nc)
        if fl is None or prof[k] <= 0:
            continue
        tf = fl * B / (prof[k] / 1e3) / 1e12
        roofline_fp64[k] = {"bound": "fp64", "achieved": round(tf, 3), "peak": fpeak, "unit": "TFLOP/s",
                            "frac": round(tf / fpeak, 4), "flops_per_launch": fl * B, "launch_ms": round(prof[k], 4),
                            "peak_source": fpeak_src}
    # HBM-bound passes of the 2D NFFT route (FFT / fold kernels): compulsory bytes of one launch
    # per problem / the live launch time.  n = coefficients per axis, n_ov = oversampled length;
    # the embedded block has n non-zero rows, so row passes touch n * n_ov entries and column
    # passes n * n_ov on one side and the full n_ov^2 grid on the other.  Folds: the per-chunk
    # partials are counted once per tile (>= one chunk per non-empty tile: a lower bound).
    roofline_passes = {}
    n_ov = int(getattr(op, "n_over", 0) or 0)
    if dim == 2 and n_ov and any(k.startswith("k2_") for k in prof):
        n_ax = int(round(Nc ** 0.5))
        ntile = ((n_ov + 11) // 12) ** 2
        R, E = 24, (2 * p if p >= 2 else 0)
        pass_bytes = {
            "k2_rows_embed_fft": 16 * Nc + 16 * n_ax * n_ov,
            "k2_cols_fft": 16 * n_ax * n_ov + 16 * n_ov * n_ov,
            "k2_fold_tiles": 16 * R * R * ntile + 16 * n_ov * n_ov,
            "k2_cols_ifft": 16 * n_ov * n_ov + 16 * n_ax * n_ov,
            "k2_rows_ifft_crop": 16 * n_ax * n_ov + 16 * Nc,
            "k2_fold_lines": 16 * 2 * E * R * ntile,
        }
        for k, bts in pass_bytes.items():
            if k in prof and prof[k] > 0 and bts > 0:
                g = bts * B / (prof[k] / 1e3) / 1e9
                roofline_passes[k] = {"bound": "hbm", "achieved": round(g, 1), "peak": peak, "unit": "GB/s",
                                      "frac": round(g / peak, 4), "bytes_per_launch": bts * B,
                                      "launch_ms": round(prof[k], 4)}
    pair_b, it_b = iteration_bytes(dim, p, M, Nc, uaxis)
    it_gbs = it_b * P / (ms_per_step / 1e3) / 1e9
    roof_iter = {"bytes_per_problem_iteration": it_b, "achieved_gbs": round(it_gbs, 2),
                 "frac": round(it_gbs / peak, 4)}

    # -------- e2e: public API from pinned host buffers (H2D of b, D2H of x inside);
    # one untimed call first (the solve workspace and its CUDA graph are built
    # once per operator), then the mean of E2E_CALLS timed calls
    b_host = data.cpu().pin_memory()
    x_host = torch.empty(B * Nc, dtype=torch.complex128).pin_memory()
    e2e_iters = CONFIG_ITERS[args.workload]
    gs_solve_host(op, b_host, x_host, e2e_iters)
    barrier(world)
    t_e = time.perf_counter()
    for _ in range(E2E_CALLS):
        xr, stats = gs_solve_host(op, b_host, x_host, e2e_iters)
    t_e = (time.perf_counter() - t_e) / E2E_CALLS
    t_e = allreduce_max(t_e, world, dev)
    e2e_value = P * e2e_iters / t_e
    h2d_call = int(b_host.numel() * 16)
    import ctypes as C
    d2h_call = int(x_host.numel() * 16 + B * C.sizeof(gs._Stats))  # solution + per-problem solve stats
    h2d, d2h = h2d_call // e2e_iters, d2h_call // e2e_iters

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(args.workload)
        out = {
            "metric": "CGLS iterations/sec (problem-iterations; T.x + T*.y pairs/sec alongside)",
            "value": round(value, 3), "unit": "problem-iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic: reference pattern generators (patterns.cpp) + seeded complex-normal coefficients",
            "config": config_for(args.workload, P, world),
            "route": route, "problems_per_rank": B,
            "l2": "inputs larger than L2 (per-point tables %.1f GB/GPU)" % (op.device_bytes / 1e9)
            if op.device_bytes > 126e6 else "L2-resident working set; back-to-back steps",
            "pairs_per_sec": round(pairs_per_sec, 3), "ms_per_pair": round(pair_ms, 4),
            "gpu_launches": int(launches),
            "roofline": roofline, "roofline_iteration": roof_iter,
            "roofline_fp64": roofline_fp64 or None,
            "roofline_passes": roofline_passes or None,
            "kernel_ms_per_pair": {k: round(v, 4) for k, v in prof.items()},
            "e2e": {"value": round(e2e_value, 3), "unit": "problem-iterations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "h2d_bytes_per_call": h2d_call, "d2h_bytes_per_call": d2h_call,
                    "steps_per_call": e2e_iters, "calls_timed": E2E_CALLS,
                    "note": "one call = the config's whole solve: gs_solve_least_squares (preamble + "
                            f"{e2e_iters} CGLS iterations, the config's count) from pinned host memory, data in and "
                            "solution + solve stats out inside the timed region; mean of the timed calls "
                            "after one untimed call; wall clock per call; per-step bytes = per-call / steps"},
            "clocks": clk, "cpu_baseline": cpu, "build_seconds": round(build_s, 1),
            "final_residual_problem0": st[0].residual,
        }
        print(json.dumps(out), flush=True)
    op.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return out


def run_gpu_sharded(args):
    """C4 across ranks: samples split into contiguous slices, one operator per
    rank, coefficient vectors replicated, NCCL allreduce of ||q||^2 and of the
    N_c-sized adjoint partial per iteration (paper_1607_04091_b200/distributed.py).
    Total work fixed -> strong scaling."""
    import torch
    import paper_1607_04091_b200 as gs
    from paper_1607_04091_b200.distributed import Communicator, ShardedSession, shard_range

    rank, world, local = dist_init(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    gen = ProductGen()
    dim, p, J, coords, mu, bw, sig = problem_inputs(args.workload, 0, gen)
    M = coords.size // dim
    lo, hi = shard_range(M, rank, world)
    my = gs.SamplingSet(dim, coords[dim * lo:dim * hi])
    op_u = gs.freq2wave(my, p, J, bandwidth=bw, device=local)
    Nc = op_u.cols()
    x_true, noise = coeffs_and_noise(0, Nc, M, sig)
    data = gs.apply_forward(op_u, torch.from_numpy(x_true).to(dev)) + torch.from_numpy(noise[lo:hi]).to(dev)
    op_u.close()
    op = gs.freq2wave(my, p, J, bandwidth=bw, weights=None if mu is None else mu[lo:hi], device=local)
    stream = torch.cuda.current_stream(dev)
    comm = Communicator.from_torch(device=local)
    L = gs.load_library()
    import ctypes as C
    L.gs_launch_count.restype = C.c_longlong
    # the library's resident sharded loop: NCCL sums of ||q||^2 and T_g* r_g on the stream
    sess = ShardedSession(op, comm, data, tolerance=1e-300, history_capacity=args.warmup + args.steps + 2,
                          stream=stream)
    sess.step(args.warmup, stream=stream)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    n0 = L.gs_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sess.step(args.steps, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = L.gs_launch_count() - n0
    clk = clocks.stop()
    ms = allreduce_max(e0.elapsed_time(e1), world, dev)
    _, st = sess.result()
    sess.close()
    comm.close()
    if rank == 0:
        peak, _ = load_peaks()
        _, it_b = iteration_bytes(dim, p, M, Nc)
        out = {"metric": "CGLS iterations/sec (problem-iterations; T.x + T*.y pairs/sec alongside)",
               "value": round(args.steps / (ms / 1e3), 3), "unit": "problem-iterations/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
               "data": "synthetic: reference pattern generators + seeded complex-normal coefficients",
               "config": config_for("c4", 1, world),
               "sharding": f"samples x{world} (library NCCL allreduce of ||q||^2 and T*r partials, "
                           f"{hi - lo} samples on rank 0)", "gpu_launches": int(launches),
               "roofline_iteration": {"bytes_per_problem_iteration": it_b,
                                      "achieved_gbs": round(it_b / (ms / args.steps / 1e3) / 1e9, 2),
                                      "frac_of_one_gpu_peak": round(it_b / (ms / args.steps / 1e3) / 1e9 / peak, 4)},
               "clocks": clk, "final_residual": st[0].residual}
        print(json.dumps(out), flush=True)
    op.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def gs_profile(op, stream):
    import ctypes as C
    import paper_1607_04091_b200 as gs
    L = gs.load_library()
    L.gs_profile_pair.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_char_p,
                                  C.POINTER(C.c_int)]
    ms = (C.c_double * 32)()
    names = C.create_string_buffer(32 * 32)
    cnt = C.c_int()
    rc = L.gs_profile_pair(op.handle, 3, C.c_void_p(stream.cuda_stream), 32, ms, names, C.byref(cnt))
    if rc:
        return {}
    out = {}
    for i in range(cnt.value):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0")[0].decode()
        out[nm] = out.get(nm, 0.0) + ms[i]
    return out


def gs_solve_host(op, b_host, x_host, iters):
    import ctypes as C
    import paper_1607_04091_b200 as gs
    L = gs.load_library()
    B = op.batch
    stats = (gs._Stats * B)()
    rc = L.gs_solve_least_squares(op.handle, b_host.data_ptr(), b_host.numel(), None, int(iters), 1e-300,
                                  x_host.data_ptr(), stats, None, None)
    gs._check(rc)
    return x_host, stats


# ------------------------------------------------------------------ CPU legs (oracle/ = test infrastructure)
def _cpu_backend():
    """(module, kind, description): the reference ITSELF when oracle/_ref/libgs_ref.so
    is present (its unmodified sources compiled with Eigen / FFTW stand-ins,
    oracle/Makefile), else the restated port (oracle/gs_oracle.cpp)."""
    import oracle
    from oracle import ref
    if os.environ.get("GS_BENCH_CPU", "") != "port" and ref.available():
        ref.lib()
        return ref, "reference", ("oracle/_ref/libgs_ref.so: the reference's own sources (proj/src/*.cpp, unmodified) "
                                  "built -O3 with an Eigen subset and a radix-2 / mixed-radix FFTW stand-in")
    oracle.lib()
    return oracle, "port", "oracle/gs_oracle.cpp, the reference algorithm restated"


def _cpu_problem(workload, b, impl):
    """The workload's problem b on the CPU implementation `impl` alone (the
    product library is never loaded by the CPU legs).  Inputs come from the
    oracle's generators (bit-identical to the reference's, tests/
    test_reference_itself.py); 2D Voronoi weights of the large configs from the
    oracle's bucketed exact clipping (the reference's O(M^2) loop is infeasible
    at 2^18-2^20 points).  Input generation is outside every timed region."""
    import oracle

    class OracleGen:
        gen_grid = staticmethod(oracle.gen_grid)
        gen_jitter = staticmethod(oracle.gen_jitter)
        gen_spiral = staticmethod(oracle.gen_spiral)

        @staticmethod
        def voronoi(dim, c, K):
            if dim == 2 and c.size > 2 * 20000:
                return oracle.voronoi_fast(dim, c, K)
            return oracle.voronoi(dim, c, K)

    dim, p, J, c, mu, bw, sig = problem_inputs(workload, b, OracleGen)
    op_u = impl.Op(dim, p, J, c, bandwidth=bw)
    x, nz = coeffs_and_noise(b, op_u.cols, op_u.rows, sig)
    data = op_u.forward(x) + nz
    del op_u
    op = impl.Op(dim, p, J, c, weights=mu, bandwidth=bw)
    return op, data


def _cpu_iter_seconds(op, data, k):
    """Seconds per CGLS iteration: (T(solve 1+k) - T(solve 1)) / k (removes the
    preamble), each solve repeated until it has run for ~0.5 s in total so that
    the microsecond-scale configs are timed over thousands of iterations."""
    def solve(n):
        t = time.perf_counter()
        op.solve(data, max_iterations=n, tolerance=1e-300)
        return time.perf_counter() - t

    probe = solve(1 + k)
    reps = int(max(1, min(2000, math.ceil(0.5 / max(probe, 1e-6)))))
    if reps == 1:
        t1, t2 = solve(1), probe
    else:
        t1 = min(sum(solve(1) for _ in range(reps)) / reps for _ in range(2))
        t2 = min(sum(solve(1 + k) for _ in range(reps)) / reps for _ in range(2))
    return max(1e-9, (t2 - t1) / k), t1, t2


def _cpu_pair_seconds(op, data):
    """Seconds per T x + T* y pair on the CPU operator (warm; repeated until ~0.5 s is timed)."""
    rng = np.random.default_rng(SEED)
    x = rng.standard_normal(op.cols) + 1j * rng.standard_normal(op.cols)

    def pair():
        t = time.perf_counter()
        op.forward(x)
        op.adjoint(data)
        return time.perf_counter() - t

    probe = pair()
    reps = int(max(1, min(5000, math.ceil(0.5 / max(probe, 1e-6)))))
    return probe if reps == 1 else min(sum(pair() for _ in range(reps)) / reps for _ in range(2))


def cpu_baseline(workload):
    """Rank 0, N=1: the reference (single-threaded, as it is) on one problem of
    the workload -- the reference itself when its library is here, else the port."""
    cpu = host_cpu()
    kind = "port"
    try:
        impl, kind, what = _cpu_backend()
        t = time.perf_counter()
        op, data = _cpu_problem(workload, 0, impl)
        build = time.perf_counter() - t
        k = 2 if workload in ("c4", "c5", "c3") else 20
        per_it, _, _ = _cpu_iter_seconds(op, data, k)
        per_pair = _cpu_pair_seconds(op, data)
        return {"value": round(1.0 / per_it, 4), "unit": "problem-iterations/s", "cores": 1, "kind": kind,
                "pairs_per_sec": round(1.0 / per_pair, 4),
                "cpu_model": cpu["model"], "physical_cores": cpu["physical_cores"],
                "sample": f"{workload.upper()} problem 0, {k} CGLS iterations (difference of solves of 1 and "
                          f"{1 + k} iterations), 1 thread, construction ({build:.1f} s) excluded; {what}"}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": "problem-iterations/s", "cores": 1, "kind": kind, "sample": f"failed: {e}"}


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path on the
    host cores (oracle/_ref, the reference itself, when present; else the
    restated port), all threads it can use -- the reference is single-threaded,
    so one problem per thread on the batched config -- same workload / metric;
    rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    impl, kind, what = _cpu_backend()
    cpu = host_cpu()
    ncpu = cpu["logical_cpus_available"]
    P = args.problems or problem_count(args.workload)
    threads = max(1, min(ncpu, P, 64 if args.workload == "c5" else 1))
    # CGLS iterations per timed solve: bounded on the large configs (seconds per iteration on a
    # core), the small ones repeat the solve until ~0.5 s has been timed (_cpu_iter_seconds)
    k = max(1, min(args.steps, 3)) if args.workload in ("c4", "c5", "c3") else 20
    rates = [0.0] * threads
    errs = []

    def work(i):
        try:
            op, data = _cpu_problem(args.workload, i, impl)
            per_it, _, _ = _cpu_iter_seconds(op, data, k)
            rates[i] = 1.0 / per_it
        except Exception as e:  # noqa: BLE001
            errs.append(str(e))

    t = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    wall = time.perf_counter() - t
    value = float(sum(rates))
    out = {"impl": "reference", "metric": "CGLS iterations/sec (problem-iterations; T.x + T*.y pairs/sec alongside)",
           "value": round(value, 4), "unit": "problem-iterations/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "c128 (f64)", "data": "synthetic (same generators and seeds as the GPU arm)",
           "config": config_for(args.workload, P, world),
           "cpu_baseline": {"value": round(value, 4), "unit": "problem-iterations/s", "cores": threads,
                            "kind": kind, "cpu_model": cpu["model"], "physical_cores": cpu["physical_cores"],
                            "sample": f"{threads} concurrent problems x {k} CGLS iterations each ({what}; "
                                      f"construction excluded); wall {wall:.0f} s"},
           "e2e": {"value": round(value, 4), "unit": "problem-iterations/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    if errs:
        out["errors"] = errs[:3]
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--problems", type=int, default=0, help="override the problem count (quick runs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard-samples", action="store_true", help="C4: sample-sharded CGLS even on one rank")
    ap.add_argument("--tensor-route", action="store_true", help="C3: the opt-in exact tensor route (default: KB-NFFT)")
    ap.add_argument("--exact-ndft", action="store_true", help="C2: the exact direct-NDFT route (default: KB-NFFT)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or args.shard_samples):
        run_gpu_sharded(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
