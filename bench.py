"""Benchmark of the randomized block matmul hot path (arXiv 2105.04940) on B200.

Default workload (BASELINE.json configs[1], "cfg2"): M 500x20000, N 20000x500
fp64, N(0,1) x lognormal(0,1.5) per column/row, K=50 unequal blocks; one step =
the configuration's sweep c in {10,20,40} blocks (W = 4000/8000/16000 columns)
x {OPL, ONC, ONMCNR two-step with c0=500}: nine approximate products, each
norm pass -> probabilities/sizes -> sampling -> gather/rescale -> C.D.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload cfg1|cfg2|cfg3]

value  = approx-product time per step (ms), device-timed with CUDA events,
         inputs resident in HBM, L2 flushed (256 MB write + 256 MB read) before every step.
e2e    = the same step through the public API with the inputs copied from
         pinned host memory and the nine C.D results read back, every step.
--impl reference times the CPU port of the reference (oracle/, kind "port")
on the host cores for the same workload.
Under torchrun each rank runs an independent replica (the sweep does not
shard; "replicas only"); value is the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads  # noqa: E402

METRIC = "approx-product time, norm-pass HBM GB/s, GEMM TC util; rel. Frobenius err"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "mc"])
    ap.add_argument("--reps", type=int, default=1000, help="replications per step (--workload mc)")
    return ap.parse_args()


# ---------------------------------------------------------------- workloads

def workload_spec(name):
    """(cfg index, data builder, list of (c_blocks, W, method, c0))."""
    if name == "cfg1":
        return 1, workloads.cfg1, [(20, 2000, m, 0) for m in ("OPL", "ONC", "UU")]
    if name == "cfg2":
        return 2, workloads.cfg2, [(cb, W, m, 500) for cb, W in zip((10, 20, 40), (4000, 8000, 16000))
                                   for m in ("OPL", "ONC", "ONMCNR")]
    if name == "cfg3":
        return 3, workloads.cfg3, [(200, 20000, "ONU", 5000)]
    raise ValueError(name)


def algorithmic(m, n, p, runs):
    norm_bytes = 8 * (m * n + n * p)
    gemm_flops = [2.0 * m * p * W for _, W, _, _ in runs]
    return norm_bytes, gemm_flops


# ---------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index=0):
        self.samples, self.proc, self.index = [], None, index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- reference arm

def cpu_cores():
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return os.cpu_count() or 1


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg, build, runs = workload_spec(args.workload)
    M, N, sizes = build()
    for _ in range(args.warmup):
        cpu_staged_step(M, N, sizes, runs, cfg)
    staged = [cpu_staged_step(M, N, sizes, runs, cfg)[0] for _ in range(args.steps)]
    times = [sum(t.values()) for t in staged]
    v = float(np.median(times))
    stages = staged[int(np.argsort(times)[len(times) // 2])]
    sample = f"{args.workload}: full step ({len(runs)} approx products), median of {args.steps}, wall clock"
    line = {
        "metric": METRIC, "value": v, "unit": "ms/step", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": args.workload, "runs": [f"{m}@W={W}" for _, W, m, _ in runs]},
        "impl": "reference",
        "cpu_baseline": {"value": v, "unit": "ms/step", "cores": cpu_cores(), "kind": "port", "sample": sample,
                         "stages_ms": stages, **cpu_info()},
        "e2e": {"value": v, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm

class L2Flush:
    """Cold L2 before a timed step: write a 256 MB buffer (> the 126 MB L2), then
    read a second 256 MB buffer so the L2 is left holding clean lines -- the
    write-back of the flush's own dirty lines is not charged to the step."""

    def __init__(self, torch):
        self.torch = torch
        self.w = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
        self.r = torch.ones(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
        self.out = torch.empty((), dtype=torch.float32, device="cuda")

    def __call__(self):
        self.w.fill_(1.0)
        self.torch.sum(self.r, dim=0, out=self.out)


def measure_dgemm_peak(torch):
    """cuBLAS float64 GEMM 8192^3 (best of 5): the measured FP64 tensor ceiling."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2105_04940_b200 as bm
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline, seeds_from_rngs

    cfg, build, runs_all = workload_spec(args.workload)
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    # N GPUs: the sweep's independent products are split over the ranks (strong scaling);
    # a single-product workload (cfg3) runs as replicas
    split = world > 1 and len(runs_all) >= world
    runs = runs_all[rank::world] if split else runs_all
    M_h, N_h, sizes = build()
    m, n = M_h.shape
    p = N_h.shape[1]
    K = len(sizes)
    Md = torch.as_tensor(M_h, device="cuda")
    Nd = torch.as_tensor(N_h, device="cuda")
    pipes = [SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs]
    group = PipelineGroup(pipes)  # the sweep's products run as concurrent graph branches
    flush = L2Flush(torch)
    stream = torch.cuda.current_stream()

    def step_seeds():
        # the call's generator work (spawn, SeedSequence hashing) on the host
        return [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs]

    def step(Mx, Nx, seeds=None):
        return group.run(Mx, Nx, seeds if seeds is not None else step_seeds())

    # correctness of the bench configuration itself (untimed), then graph capture
    first = [o.cpu().numpy() for o in step(Md, Nd)]
    for pipe in pipes:
        pipe.check()
    parity = golden_parity(args.workload, runs, pipes, first)
    group.capture(Md, Nd)
    for _ in range(args.warmup):
        step(Md, Nd)
    torch.cuda.synchronize()

    # ---- device-timed steps (inputs resident, L2 flushed before each step)
    n_launch0 = _lib.launches()
    times = []
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush()
            seeds = step_seeds()  # host-side inputs of the step, ready before it starts (as M and N)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(Md, Nd, seeds)
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    # eager launches (none when every pipeline replays its CUDA graph) + graph-contained kernels
    launches = (_lib.launches() - n_launch0) // args.steps + group.graph_launches
    ms = [a.elapsed_time(b) for a, b in times]
    ms_step = float(np.mean(ms))
    if world > 1:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())

    # ---- e2e through the public API with host buffers (pinned) every step: one graph
    # from pinned M, N to pinned products -- chunked H2D transfer with the norm pass
    # and OPL's segmented square sums behind it (PipelineGroup.capture_host)
    M_pin = torch.from_numpy(M_h).pin_memory()
    N_pin = torch.from_numpy(N_h).pin_memory()
    Mx, Nx = torch.empty_like(Md), torch.empty_like(Nd)
    outs_h = [torch.empty((m, p), dtype=torch.float64).pin_memory() for _ in runs]
    host_group = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs],
                               joint=os.environ.get("BMM_E2E_JOINT", "0") == "1")  # per-branch GEMMs measured faster end to end
    host_group.capture_host(Mx, Nx, M_pin, N_pin, outs_h,
                            [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs],
                            n_chunks=int(os.environ.get("BMM_E2E_CHUNKS", "8")))
    e2e = []
    for it in range(args.warmup + args.steps):
        seeds = [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_group.run_host(seeds)
        torch.cuda.synchronize()
        if it >= args.warmup:
            e2e.append((time.perf_counter() - t0) * 1e3)
    ref_outs = group.run(Md, Nd, [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K)
                                  for cb, W, meth, c0 in runs])
    for o, h in zip(ref_outs, outs_h):  # the streamed graph computes the same products
        # (bit-identical draws and sketches; the resident group's joint batched GEMM splits
        # the inner sum differently from the per-branch GEMMs of the streamed graph)
        o = o.cpu()
        same = (torch.equal(o, h) if group.joint == host_group.joint
                else bool(((o - h).norm() <= 1e-13 * o.norm()).item()))
        if not same:
            raise RuntimeError("streamed end-to-end products differ from the resident run: rel "
                               f"{float((o - h).norm() / o.norm()):.3e}, finite {bool(torch.isfinite(o).all())} "
                               f"{bool(torch.isfinite(h).all())}, joint {group.joint}/{host_group.joint}")
    latency_ms = float(np.mean(e2e))
    # steady state: a second instance of the streamed graph alternates with the first on two
    # streams, so one step's host->device transfer overlaps the previous step's work; every
    # step still copies its inputs in and its products out
    Mx2, Nx2 = torch.empty_like(Md), torch.empty_like(Nd)
    outs_h2 = [torch.empty((m, p), dtype=torch.float64).pin_memory() for _ in runs]
    host_group2 = PipelineGroup([SketchPipeline(m, n, p, sizes, W, meth, c0=c0) for _, W, meth, c0 in runs],
                                joint=host_group.joint)
    host_group2.capture_host(Mx2, Nx2, M_pin, N_pin, outs_h2,
                             [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs],
                             n_chunks=int(os.environ.get("BMM_E2E_CHUNKS", "8")))
    lanes = [(host_group, torch.cuda.Stream()), (host_group2, torch.cuda.Stream())]
    ksteps = max(10, args.steps)
    for it in range(2 + ksteps):
        if it == 2:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
        g_, s_ = lanes[it % 2]
        seeds = [seeds_from_rngs(meth, [workloads.sample_rng(cfg, cb)], K) for cb, W, meth, c0 in runs]
        with torch.cuda.stream(s_):
            g_.run_host(seeds)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / ksteps
    if not all(torch.equal(a, b) for a, b in zip(outs_h, outs_h2)):
        raise RuntimeError("pipelined end-to-end products differ")
    h2d = M_h.nbytes + N_h.nbytes
    d2h = len(runs) * m * p * 8
    # the drop-in API on numpy inputs, call for call as the reference's bench loop
    # (bench.py:209-245): allocate_* + estimate_product (or estimate_product_two_step);
    # every call uploads M and N and returns the SketchPair / SampleLog records to the host
    part = bm.BlockPartition(sizes)
    dropin = []
    for it in range(1 + min(args.steps, 3)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for cb, W, meth, c0 in runs:
            rng = workloads.sample_rng(cfg, cb)
            if meth in ("ONU", "ONMCNR"):
                bm.estimate_product_two_step(M_h, N_h, part, W, c0, rng,
                                             pilot="uniform" if meth == "ONU" else "norm")
            else:
                fn = {"OPL": bm.allocate_optimal, "ONC": bm.allocate_by_score_sums, "UU": None}[meth]
                plan = fn(M_h, N_h, part, W) if fn is not None else bm.allocate_uniform(part, W)
                bm.estimate_product(M_h, N_h, plan, rng)
        torch.cuda.synchronize()
        if it >= 1:
            dropin.append((time.perf_counter() - t0) * 1e3)

    # ---- roofline of the dominant kernels, timed live (events around their launches)
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peak.get("hbm_gbs", 6650.0))
    norm_bytes, gemm_flops = algorithmic(m, n, p, runs)
    kt = kernel_times(torch, bm, pipes, runs, Md, Nd, cfg, K, flush, group)
    dgemm_peak = measure_dgemm_peak(torch)
    gemm_ms = kt["gemm_ms"]
    # executed flops: 2 m p K over the distinct drawn columns the GEMM contracts
    gemm_flops = [2.0 * m * p * kd for kd in kt["gemm_k"]]
    gemm_achieved = sum(gemm_flops) / (sum(gemm_ms) * 1e-3) / 1e12
    norms_achieved = norm_bytes / (kt["norms_ms"] * 1e-3) / 1e9
    large = norms_large(torch)

    # errors of the W=16000 ONC product vs the exact product (verification, untimed)
    from paper_2105_04940_b200.analysis import sq_diff
    exact = bm.multiply_exact(Md, Nd)
    idx = len(runs) - 1  # the widest product of the sweep
    meth_e = runs[idx][2]
    CD = step(Md, Nd)[idx]
    err_sq, ref_sq = sq_diff(exact, CD)
    fro_m = np.linalg.norm(M_h)
    fro_n = np.linalg.norm(N_h)

    # dominant kernel by device time per step: OPL's segmented square sums when the sweep has OPL
    # products (3 x 2 m p n flops at cfg2), else the sampled GEMM
    gemm_step_ms = sum(gemm_ms)
    roofline_main = None
    roofline_gemm_i8 = None
    if all(e == "i8" for e in kt["gemm_engine"]):
        i8_peak = 2.0 * float(peak.get("bf16_tflops", 1635.9))
        i8_ops = sum(36.0 * f for f in gemm_flops)
        roofline_gemm_i8 = {
            "bound": "tensor", "kernel": "bmm_gemm_i8_gather (C.D: sketch gather fused into the Ozaki digit split, "
                                        "int8 tcgen05 contraction, split-K reduction)",
            "achieved": i8_ops / (sum(gemm_ms) * 1e-3) / 1e12, "peak": i8_peak, "unit": "TOPS (int8)",
            "frac": i8_ops / (sum(gemm_ms) * 1e-3) / 1e12 / i8_peak,
            "peak_source": "dense int8 = 2 x MEASURED_PEAKS bf16_tflops (burst)",
            "algorithmic": "36 x 2*m*p*K int8 ops over the distinct drawn columns; the time includes the gather "
                           "and digit split",
            "f64_equivalent_tflops": gemm_achieved, "dgemm_peak_tflops": dgemm_peak,
            "cublas_same_shapes_tflops": sum(gemm_flops) / (sum(kt["cublas_same_shape_ms"]) * 1e-3) / 1e12,
            "traffic": None}
    roofline_segsq = None
    if "segsq_ms" in kt and kt["segsq_engine"] == "i8":
        # OPL g_k^2 on the int8 tensor cores: 36 int8 digit-plane products (levels t+u <= 7 of
        # 8 x 8 planes) per float64 multiply-add, 2*m*p*n float64 flops per launch
        i8_ops = 36 * 2.0 * m * p * n
        i8_peak = 2.0 * float(peak.get("bf16_tflops", 1635.9))
        i8_achieved = i8_ops / (kt["segsq_contract_ms"] * 1e-3) / 1e12
        roofline_main = {"bound": "tensor", "kernel": "oz_segsq_kernel (OPL g_k^2 = ||M^k N_k||_F^2: int8 tcgen05 "
                                                     "contraction of the Ozaki digit planes)",
                         "achieved": i8_achieved, "peak": i8_peak, "unit": "TOPS (int8)",
                         "frac": i8_achieved / i8_peak,
                         "peak_source": "dense int8 = 2 x MEASURED_PEAKS bf16_tflops (burst): the same tcgen05 "
                                        "cycles per dispatch at K=32 int8 vs K=16 bf16",
                         "algorithmic": "36 x 2*m*p*n int8 ops per launch (8 digit planes per operand, "
                                        "products with t+u <= 7)",
                         "launch_ms": kt["segsq_contract_ms"],
                         "share_of_step_device_ms": kt["segsq_ms"] * kt["segsq_per_step"],
                         "segsq_total_ms": kt["segsq_ms"], "split_ms": kt["segsq_split_ms"],
                         "f64_equivalent_tflops": 2.0 * m * p * n / (kt["segsq_ms"] * 1e-3) / 1e12,
                         "f64_equivalent_frac_of_dgemm": 2.0 * m * p * n / (kt["segsq_ms"] * 1e-3) / 1e12 / dgemm_peak,
                         "traffic": None,
                         "traffic_note": "see profiles/ (ncu --set full of oz_segsq_kernel)"}
        # the dominant kernel by device time per step: the contraction (3 launches at cfg2) or
        # the nine sampled DMMA GEMMs
        if kt["segsq_contract_ms"] * kt["segsq_per_step"] < gemm_step_ms:
            roofline_segsq, roofline_main = roofline_main, None
    elif "segsq_ms" in kt and kt["segsq_ms"] * kt["segsq_per_step"] > gemm_step_ms:
        seg_flops = 2.0 * m * p * n
        seg_achieved = seg_flops / (kt["segsq_ms"] * 1e-3) / 1e12
        roofline_main = {"bound": "tensor", "kernel": "segsq_f64_kernel (OPL g_k^2 = ||M^k N_k||_F^2, DMMA)",
                         "achieved": seg_achieved, "peak": dgemm_peak, "unit": "TFLOP/s",
                         "frac": seg_achieved / dgemm_peak,
                         "peak_source": "cuBLAS dgemm 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64)",
                         "algorithmic": "2*m*p*n flops per launch", "launch_ms": kt["segsq_ms"],
                         "share_of_step_device_ms": kt["segsq_ms"] * kt["segsq_per_step"],
                         "traffic": 164780800 if (m, n, p) == (500, 20000, 500) else None,
                         "traffic_note": "dram__bytes_read+write per launch, ncu --set full "
                                         "(profiles/r1e_ncu_full_summary.csv): 0.160 GB + 4.7 MB = M + N read once"}
    line = {
        "metric": METRIC, "value": ms_step, "unit": "ms/step", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": args.workload, "m": m, "n": n, "p": p, "K": K,
                   "runs": [f"{meth}@W={W}" for _, W, meth, _ in runs_all], "l2": "flushed (256 MB write, then 256 MB read) before each step",
                   "parallelism": (f"the sweep's {len(runs_all)} products split over {world} GPUs" if split else
                                   f"replicas x{world}" if world > 1 else "1 GPU")},
        "scaling": "strong" if split else "weak",
        "e2e": {"value": e2e_ms, "unit": "ms/step", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "latency_ms": latency_ms,
                "api": "PipelineGroup.capture_host/run_host: pinned host M, N -> pinned host products (one graph)",
                "mode": "steady state of consecutive steps, two step instances alternating on two streams "
                        "(transfer of step i+1 overlaps the work of step i); latency_ms: one step alone"},
        "e2e_dropin_api": {"value": float(np.mean(dropin)), "unit": "ms/step",
                           "api": "allocate_* + estimate_product / estimate_product_two_step on numpy inputs, one "
                                  "call per product as the reference's bench loop (uploads M and N per call, "
                                  "returns C, D and the sample log to the host)"},
        "gpu_launches": int(launches),
        "roofline": roofline_main,
        "roofline_gemm": roofline_gemm_i8 if roofline_gemm_i8 is not None else
                    {"bound": "tensor", "kernel": "gemm_f64_kernel (C.D, DMMA" + (
                        ", one batched launch per sketch width over the sweep's products)" if group.joint else ")"),
                     "achieved": gemm_achieved,
                     "peak": dgemm_peak, "unit": "TFLOP/s", "frac": gemm_achieved / dgemm_peak,
                     "peak_source": "cuBLAS dgemm 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64)",
                     "cublas_same_shapes_tflops": sum(gemm_flops) / (sum(kt["cublas_same_shape_ms"]) * 1e-3) / 1e12,
                     "flops_note": "executed 2*m*p*K over the distinct drawn columns (gemm_k); the sketch "
                                   "width W counts duplicates, which the compressed sketch folds into scales",
                     "traffic": (285300000 if group.joint else 35511000) if (m, p) == (500, 500) else None,
                     "traffic_note": ("ncu --set full of the three per-width joint launches and their split-K "
                                      "reductions (profiles/r1n_ncu_joint_gemm.csv, tools/joint_gemm_probe.py): "
                                      "231 MB in the GEMMs = the nine gathered C and D read once (+ partials), "
                                      "54 MB in the reductions; DMMA pipe 77-82% active")
                                     if group.joint else
                                     "ncu --set full, W=16000 ONC launch (profiles/r1e_ncu_full_summary.csv): "
                                     "35.5 MB = the gathered C and D read once"},
        "roofline_segsq": roofline_segsq,
        "roofline_norms": {"bound": "hbm", "kernel": "colsq/rowsq (K1)", "achieved": norms_achieved,
                           "peak": hbm_peak, "unit": "GB/s", "frac": norms_achieved / hbm_peak,
                           "algorithmic_bytes": norm_bytes,
                           "note": "160 MB per pass: latency-bound size (SURVEY §7 K1); see roofline_norms_large"},
        "roofline_norms_large": dict(large, peak=hbm_peak, frac=large["achieved"] / hbm_peak),
        "kernel_ms": {k: v for k, v in kt.items() if k != "gemm_ms"} | {"gemm_ms": gemm_ms},
        "rel_err_baseline_metric": float(np.sqrt(err_sq) / (fro_m * fro_n)),
        "rel_err_reference_metric": float(np.sqrt(err_sq / ref_sq)),
        "clocks": clocks.summary(),
    }
    if line["roofline"] is None:
        line["roofline"] = line["roofline_gemm"]
    if rank == 0:
        if world == 1:
            cb, oracle_out = cpu_baseline(M_h, N_h, sizes, runs, cfg, args)
            line["cpu_baseline"] = cb
            parity.update(oracle_parity(runs, pipes, first, oracle_out))
        line["parity"] = parity
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def kernel_times(torch, bm, pipes, runs, Md, Nd, cfg, K, flush, group=None):
    """Per-kernel device times with CUDA events on the launching stream."""
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.pipeline import seeds_from_rngs
    st = _lib.stream_ptr()
    lib = _lib.load()
    out = {"gemm_ms": []}
    m, n = Md.shape
    p = Nd.shape[1]
    # norm pass alone (L2 flushed first)
    pipe = pipes[0]
    reps = []
    for _ in range(5):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.bmm_norms(0, Md.data_ptr(), m, n, n, 0, Nd.data_ptr(), p, p, 0, 1, 0, pipe.colsq.data_ptr(),
                      pipe.rowsq.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        reps.append(e0.elapsed_time(e1))
    out["norms_ms"] = float(np.median(reps))
    # OPL's segmented square sums g_k^2 (K7), once per OPL product
    opl = [pipe for (cb, W, meth, c0), pipe in zip(runs, pipes) if meth == "OPL"]
    if opl:
        pipe = opl[0]
        reps, parts = [], []
        for _ in range(5):
            flush()
            if pipe.seg_engine == "i8":
                ms3 = (ctypes.c_float * 3)()
                _lib.call("bmm_segsq_i8_timed", 0, Md.data_ptr(), n, 0, Nd.data_ptr(), p, 0, m, p, n,
                          pipe.offsets.data_ptr(), pipe.K, 0, 1, pipe.gsq.data_ptr(), pipe.ws_seg.data_ptr(),
                          pipe.ws_seg.numel(), st, ms3)
                parts.append(list(ms3))
                reps.append(sum(ms3))
                continue
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            lib.bmm_segsq_f64(Md.data_ptr(), n, 0, Nd.data_ptr(), p, 0, m, p, pipe.offsets.data_ptr(), pipe.K, 0, 1,
                              pipe.gsq.data_ptr(), pipe.ws_seg.data_ptr(), pipe.ws_seg.numel(), st)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        out["segsq_ms"] = float(np.median(reps))
        out["segsq_per_step"] = len(opl)
        out["segsq_engine"] = pipe.seg_engine
        if parts:
            med = np.median(np.asarray(parts), axis=0)
            out["segsq_split_ms"], out["segsq_contract_ms"], out["segsq_reduce_ms"] = (float(x) for x in med)
    # the sampled GEMM of each run (C, D already gathered by the last step): over the
    # distinct drawn columns when the pipeline compresses the sketch (k_count on device)
    out["gemm_k"] = []
    joint = group is not None and getattr(group, "joint", False)
    if joint:
        # one batched DMMA GEMM contracts every product of the step (PipelineGroup joint mode)
        kk = {}
        for jg in group._jgroups:
            for i, x in zip(jg["idx"], jg["k"].cpu().numpy()):
                kk[i] = int(x)
        out["gemm_k"] = [kk[i] for i in range(len(pipes))]
        reps = []
        for _ in range(5):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            group._joint_gemm()
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        out["gemm_ms"].append(float(np.median(reps)))
        out["gemm_joint"] = (f"{len(group._jgroups)} batched GEMMs (one per sketch width) over the {len(pipes)} "
                             "products (pooled operands)")
    for (cb, W, meth, c0), pipe in zip(runs, pipes):
        if joint:
            break
        kd = int(pipe.k_count[0].item()) if pipe.compress else W
        out["gemm_k"].append(kd)

        def gemm():
            if getattr(pipe, "gemm_engine", "dmma") == "i8":
                pipe.contract(Md, Nd, st)
            elif pipe.compress:
                lib.bmm_gemm_f64_dk(pipe.C.data_ptr(), W, m * W, pipe.D.data_ptr(), p, W * p, m, p, W,
                                    pipe.k_count.data_ptr(), 1, pipe.CD.data_ptr(), p, m * p, pipe.ws_gemm.data_ptr(),
                                    pipe.ws_gemm.numel(), st)
            else:
                lib.bmm_gemm_f64(pipe.C.data_ptr(), W, m * W, pipe.D.data_ptr(), p, W * p, m, p, W, 1,
                                 pipe.CD.data_ptr(), p, m * p, pipe.ws_gemm.data_ptr(), pipe.ws_gemm.numel(), st)
        reps = []
        for _ in range(5):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gemm()
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        out["gemm_ms"].append(float(np.median(reps)))
    # context: cuBLAS DGEMM on the same operands (reference point only; not on the product path)
    out["cublas_same_shape_ms"] = []
    out["gemm_engine"] = [getattr(pipe, "gemm_engine", "dmma") for pipe in pipes]
    for (cb, W, meth, c0), pipe, kd in zip(runs, pipes, out["gemm_k"]):
        if hasattr(pipe, "C"):
            Wc = pipe._joint or W  # pooled operands (joint group) have the pool's row stride
            C, D = pipe.C.view(m, Wc)[:, :kd], pipe.D.view(Wc, p)[:kd]
        else:  # the i8 engine gathers inside its split: build C, D for the cuBLAS reference point
            col, sc = (pipe.k_column, pipe.k_scale) if pipe.compress else (pipe.column, pipe.scale)
            C = Md[:, col[:kd]] * sc[:kd]
            D = Nd[col[:kd], :] * sc[:kd, None]
        torch.matmul(C, D)
        reps = []
        for _ in range(5):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(C, D)
            e1.record()
            torch.cuda.synchronize()
            reps.append(e0.elapsed_time(e1))
        out["cublas_same_shape_ms"].append(float(np.median(reps)))
    return out


def norms_large(torch, problems=1024):
    """K1 on a bandwidth-scale input: `problems` config-5 problems (float32,
    256x4096 and 4096x256 each; 8.6 GB at 1024), median of 3 timed launches."""
    from paper_2105_04940_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(workloads.ROOT)
    m, n, p = 256, 4096, 256
    M = torch.randn((problems, m, n), generator=g, device="cuda", dtype=torch.float32)
    N = torch.randn((problems, n, p), generator=g, device="cuda", dtype=torch.float32)
    cs = torch.empty(problems * n, dtype=torch.float64, device="cuda")
    rs = torch.empty(problems * n, dtype=torch.float64, device="cuda")
    lib, st = _lib.load(), _lib.stream_ptr()
    reps = []
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.bmm_norms(1, M.data_ptr(), m, n, n, m * n, N.data_ptr(), p, p, n * p, problems, 0, cs.data_ptr(),
                      rs.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        reps.append(e0.elapsed_time(e1))
    ms = float(np.median(reps[1:]))
    nbytes = 4 * problems * (m * n + n * p)
    del M, N
    torch.cuda.empty_cache()
    return {"bound": "hbm", "kernel": "colsq/rowsq (K1)", "input": f"{problems} config-5 problems (float32)",
            "algorithmic_bytes": nbytes, "ms": ms, "achieved": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s"}


def cpu_staged_step(M, N, sizes, runs, cfg):
    """One step of the reference path with the oracle port (NumPy + BLAS), timed
    per stage as SURVEY.md §8(d5) asks: the norm pass (colsq, rowsq, probabilities),
    the plan (g_k for OPL, the pilot for two-step, integerize), the sample (child
    streams, draws, gather of C and D) and C @ D.  Returns ({stage: ms}, outputs)."""
    from oracle import blockmm_oracle as O
    t = {"norms": 0.0, "plan": 0.0, "sample": 0.0, "gemm": 0.0}
    outs = []
    K = len(sizes)

    def clock(key, fn):
        t0 = time.perf_counter()
        r = fn()
        t[key] += (time.perf_counter() - t0) * 1e3
        return r

    for cb, W, meth, c0 in runs:
        rng = workloads.sample_rng(cfg, cb)
        # the reference recomputes the norm pass inside every allocator (plan.py:165-189)
        cs, rs, probs, s = clock("norms", lambda: O.instance_stats(M, N, sizes))
        if meth in ("ONU", "ONMCNR"):
            pilot_sq, _, _, main_rng = clock("plan", lambda: O.two_step_pilot(M, N, sizes, c0, meth, rng, probs, s))
            budgets, _ = clock("plan", lambda: O.plan_budgets("TWO_STEP", sizes, W, s=s, aux_sq=pilot_sq))
            srng = main_rng
        elif meth == "OPL":
            gsq = clock("plan", lambda: O.block_product_sq(M, N, sizes))
            budgets, _ = clock("plan", lambda: O.plan_budgets("OPL", sizes, W, s=s, aux_sq=gsq))
            srng = rng
        elif meth == "ONC":
            budgets, _ = clock("plan", lambda: O.plan_budgets("ONC", sizes, W, s=s))
            srng = rng
        else:  # UU
            probs = np.concatenate([np.full(nk, 1.0 / nk) for nk in sizes])
            budgets, _ = clock("plan", lambda: O.plan_budgets("UU", sizes, W))
            srng = rng
        cols, _, scale, C, D = clock("sample", lambda: O.sketch(M, N, sizes, probs, budgets, srng.spawn(K)))
        CD = clock("gemm", lambda: C @ D)
        outs.append({"budgets": budgets, "columns": cols, "scale": scale, "CD": CD})
    return t, outs


def cpu_baseline(M, N, sizes, runs, cfg, args, reps=5):
    """The CPU port of the step at all BLAS threads and at 1 thread (medians of
    `reps`), with the stage split and the host description."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    res, out = {}, None
    for label, lim in (("all", None), ("1", 1)):
        ctx = threadpool_limits(limits=lim) if (threadpool_limits and lim) else None
        if ctx is not None:
            ctx.__enter__()
        try:
            runs_t = []
            for _ in range(reps):
                tt, o = cpu_staged_step(M, N, sizes, runs, cfg)
                runs_t.append(tt)
                out = out or o
        finally:
            if ctx is not None:
                ctx.__exit__(None, None, None)
        tot = [sum(r.values()) for r in runs_t]
        med = int(np.argsort(tot)[len(tot) // 2])
        res[label] = {"ms": float(np.median(tot)), "stages_ms": runs_t[med]}
    cb = {"value": res["all"]["ms"], "unit": "ms/step", "cores": cpu_cores(), "kind": "port",
          "value_1thread": res["1"]["ms"], "stages_ms": res["all"]["stages_ms"],
          "stages_ms_1thread": res["1"]["stages_ms"], "median_of": reps,
          "sample": f"{args.workload}: full step ({len(runs)} approx products) with oracle/blockmm_oracle.py "
                    f"(NumPy + BLAS); medians of {reps} at all BLAS threads and at 1 thread; wall clock",
          **cpu_info()}
    return cb, out


def golden_parity(workload, runs, pipes, outs):
    """Untimed: the benched products against the reference's own outputs
    (tests/golden/cfg2.npz, written by running the reference): budgets, draws
    and scales bit-exact, C.D (every 7th row/column and the Frobenius norm)
    within 1e-12."""
    path = ROOT / "tests" / "golden" / f"{workload}.npz"
    if workload != "cfg2" or not path.exists():
        return {}
    g = np.load(path)
    worst = 0.0
    for (cb, W, meth, c0), pipe, CD in zip(runs, pipes, outs):
        key = f"{meth}_{W}"
        if not (np.array_equal(pipe.budgets_host()[0], g[key + "_budgets"])
                and np.array_equal(pipe.columns_host()[0], g[key + "_columns"])
                and np.array_equal(pipe.scales_host()[0], g[key + "_scale"])):
            raise RuntimeError(f"{workload} {key}: budgets / draws differ from the reference golden")
        sub = g[key + "_CDsub"]
        e = max(float(np.linalg.norm(CD[::7, ::7] - sub) / np.linalg.norm(sub)),
                abs(float(np.linalg.norm(CD)) - float(g[key + "_CDfrob"])) / float(g[key + "_CDfrob"]))
        if e > 1e-12:
            raise RuntimeError(f"{workload} {key}: C.D rel err {e:.2e} vs the reference golden")
        worst = max(worst, e)
    return {"golden_ok": True, "golden": str(path.relative_to(ROOT)), "golden_cd_max_rel_err": worst}


def oracle_parity(runs, pipes, outs, oracle_outs):
    """Untimed: the benched products against the CPU baseline's own oracle run
    of the same step (budgets, draws, scales bit-exact; C.D within 1e-12)."""
    worst = 0.0
    for (cb, W, meth, c0), pipe, CD, ref in zip(runs, pipes, outs, oracle_outs):
        if not (np.array_equal(pipe.budgets_host()[0], ref["budgets"])
                and np.array_equal(pipe.columns_host()[0], ref["columns"])
                and np.array_equal(pipe.scales_host()[0], ref["scale"])):
            raise RuntimeError(f"{meth}@W={W}: budgets / draws differ from the oracle")
        e = float(np.linalg.norm(CD - ref["CD"]) / np.linalg.norm(ref["CD"]))
        if e > 1e-12:
            raise RuntimeError(f"{meth}@W={W}: C.D rel err {e:.2e} vs the oracle")
        worst = max(worst, e)
    return {"ok": True, "oracle_cd_max_rel_err": worst,
            "checked": "budgets, every draw and scale bit-exact; C.D within 1e-12 (float64)"}


# ---------------------------------------------------------------- float32 device workloads (cfg4, cfg5)

def device_data(torch, name, problems=None):
    """Seeded float32 instances generated on the GPU (numpy would take minutes
    for 2 x 8.6e9 normals); distributions per SURVEY.md §8(d).  cfg5 is
    generated in chunks of 256 problems, each chunk from its own seed, so a rank
    of a sharded run regenerates exactly its problems (`problems` = (lo, hi))."""
    if name == "cfg5":
        B, m, n, p, K, CH = 4096, 256, 4096, 256, 64, 256
        lo, hi = problems or (0, B)
        M = torch.empty((hi - lo, m, n), dtype=torch.float32, device="cuda")
        N = torch.empty((hi - lo, n, p), dtype=torch.float32, device="cuda")
        for c in range(lo // CH, (hi + CH - 1) // CH):
            g = torch.Generator(device="cuda").manual_seed(workloads.ROOT * 1000 + 50000 + c)
            Mc = torch.empty((CH, m, n), dtype=torch.float32, device="cuda").normal_(generator=g)
            Mc.mul_(torch.randn((CH, 1, n), generator=g, device="cuda").exp_())
            Nc = torch.empty((CH, n, p), dtype=torch.float32, device="cuda").normal_(generator=g)
            Nc.mul_(torch.randn((CH, n, 1), generator=g, device="cuda").exp_())
            a, b = max(lo, c * CH), min(hi, c * CH + CH)
            M[a - lo:b - lo] = Mc[a - c * CH:b - c * CH]
            N[a - lo:b - lo] = Nc[a - c * CH:b - c * CH]
            del Mc, Nc
        return M, N, (n // K,) * K, hi - lo
    M, N = cfg4_shard(torch, (0, 16384), (0, 16384))
    return M, N, (262144 // 4096,) * 4096, 1


def cfg4_shard(torch, rows, cols):
    """Rows `rows` of config 4's M and columns `cols` of its N, float32 on the
    GPU.  Generation is chunk-seeded (1024-row chunks of M, 16384-row chunks of
    N), so every rank of a sharded run regenerates exactly its slice of the
    same global instance; per-block scales U[0.1, 10] for M^k and N_k."""
    m, n, p, K = 16384, 262144, 16384, 4096
    g = torch.Generator(device="cuda").manual_seed(workloads.ROOT + 4)
    cs = (torch.rand(K, generator=g, device="cuda") * 9.9 + 0.1).repeat_interleave(n // K)
    rs = (torch.rand(K, generator=g, device="cuda") * 9.9 + 0.1).repeat_interleave(n // K)
    r0, r1 = rows
    c0, c1 = cols
    M = torch.empty((r1 - r0, n), dtype=torch.float32, device="cuda")
    N = torch.empty((n, c1 - c0), dtype=torch.float32, device="cuda")
    for ch in range(r0 // 1024, (r1 + 1023) // 1024):
        gc = torch.Generator(device="cuda").manual_seed(workloads.ROOT * 1000 + 40000 + ch)
        blk = torch.empty((1024, n), dtype=torch.float32, device="cuda").normal_(generator=gc).mul_(cs)
        a, b = max(r0, ch * 1024), min(r1, ch * 1024 + 1024)
        M[a - r0:b - r0] = blk[a - ch * 1024:b - ch * 1024]
        del blk
    for ch in range(n // 16384):
        gc = torch.Generator(device="cuda").manual_seed(workloads.ROOT * 1000 + 41000 + ch)
        blk = torch.empty((16384, p), dtype=torch.float32, device="cuda").normal_(generator=gc)
        N[ch * 16384:(ch + 1) * 16384] = blk[:, c0:c1] * rs[ch * 16384:(ch + 1) * 16384, None]
        del blk
    return M, N


def run_cfg4_sharded(args):
    """Config 4 with M's rows and N's columns sharded over the torchrun group
    (SURVEY.md §8(e), strong scaling): the same step as run_cfg4 (OPL, ONC,
    SSM over one instance) through distributed.ShardedApproxProduct.  The only
    exchanges are the exact norm pass (chained colsq stages, tree-combined
    rowsq: plans and draws bit-identical to one GPU) and the K-length g_k^2
    partials.  value = ms per step of the whole problem, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2105_04940_b200.distributed import ShardLayout, ShardedApproxProduct

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}")
    m, n, p, K = 16384, 262144, 16384, 4096
    sizes = (n // K,) * K
    L = ShardLayout(world, rank, m, n, p)
    M, N = cfg4_shard(torch, L.rows, L.cols)
    sh = ShardedApproxProduct(L, sizes, [(meth, w) for meth, w, _ in CFG4_RUNS], dtype=torch.float32)
    tiles = sh.run(M, N, cfg4_seeds(K))
    sh.check()
    # every rank drew the single-GPU sample: compare the draws across ranks (identical bits)
    cols = torch.cat([q.column[:q.W] if q.method != "SSM" else q.blk for q in sh.pipes]).contiguous()
    allc = [torch.empty_like(cols) for _ in range(world)]
    dist.all_gather(allc, cols)
    same_draws = all(torch.equal(c, cols) for c in allc)
    for _ in range(args.warmup):
        sh.run(M, N, cfg4_seeds(K))
    torch.cuda.synchronize()
    from paper_2105_04940_b200 import _lib as _l
    times = []
    n_l0 = _l.launches()
    with ClockSampler(local) as clocks:
        dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            seeds = cfg4_seeds(K)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sh.run(M, N, seeds)
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
        dist.barrier()
    launches = (_l.launches() - n_l0) // max(1, args.steps)
    ms = torch.tensor([float(np.mean([a.elapsed_time(b) for a, b in times]))], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    # e2e: this rank's shard from pinned host memory, its tiles back, every step (skipped
    # when the node's RAM cannot pin every rank's shard)
    import psutil
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    need = (M.numel() + N.numel() + sum(t.numel() for t in tiles)) * 4 * local_world
    can = torch.tensor([1.0 if psutil.virtual_memory().available > need + (16 << 30) else 0.0], device="cuda")
    dist.all_reduce(can, op=dist.ReduceOp.MIN)
    if can.item() < 1.0:
        e2e_line = {"value": None, "unit": "ms/step", "skipped": "host RAM too small to pin every rank's shard"}
        ms_e2e = None
    else:
        e2e_line = None
    M_pin = torch.empty(M.shape, dtype=M.dtype).pin_memory() if e2e_line is None else None
    N_pin = torch.empty(N.shape, dtype=N.dtype).pin_memory() if e2e_line is None else None
    if e2e_line is None:
        M_pin.copy_(M)
        N_pin.copy_(N)
    outs = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in tiles] if e2e_line is None else []
    e2e = []
    for it in range(1 + args.steps if e2e_line is None else 0):
        seeds = cfg4_seeds(K)
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        M.copy_(M_pin, non_blocking=True)
        N.copy_(N_pin, non_blocking=True)
        for o, t in zip(outs, sh.run(M, N, seeds)):
            o.copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        if it >= 1:
            e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_t = torch.tensor([float(np.mean(e2e)) if e2e else 0.0], device="cuda")
    dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": float(ms.item()), "unit": "ms/step", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(ms.item()), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (fp16 split-operand tensor contraction on CTA pairs, f64 norms/plan)",
            "data": "synthetic (chunk-seeded on device: every rank regenerates exactly its slice)",
            "config": {"workload": "cfg4", "grid": list(L.grid), "m": m, "n": n, "p": p, "K": K, "block": 64,
                       "runs": ["OPL@W=32768", "ONC@W=32768", "SSM@draws=512"],
                       "parallelism": f"M rows x N cols over {world} GPUs ({L.grid[0]}x{L.grid[1]}); exact norm "
                                      "exchange + g_k^2 partials (NCCL all-gather)",
                       "l2": "inputs >> L2"},
            "draws_identical_on_all_ranks": bool(same_draws),
            "gpu_launches": int(launches),
            "e2e": e2e_line if e2e_line is not None else
                   {"value": float(e2e_t.item()), "unit": "ms/step",
                    "h2d_bytes_per_step": int(M.numel() * 4 + N.numel() * 4) * world,
                    "d2h_bytes_per_step": int(sum(t.numel() for t in tiles) * 4) * world,
                    "api": "ShardedApproxProduct.run on each rank's shard copied from pinned host memory"},
            "clocks": clocks.summary()}), flush=True)
    dist.destroy_process_group()
    return 0


def relaunch_distributed(args):
    """`--gpus N` (N > 1) outside torchrun: start N ranks of this same command
    with torch.distributed.run on 127.0.0.1 (NCCL INFO logs to stderr so the
    ranks can be counted)."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_FILE=os.environ.get("NCCL_DEBUG_FILE", "/dev/stderr"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def cfg5_cpu_baseline(pipe, CD, Md, Nd, sizes, W, keys, sample=16):
    """Config 5 on the host: the oracle port (NumPy + BLAS) over `sample`
    problems spread across the batch, per-problem stages timed and scaled to
    4096 problems (all BLAS threads and 1 thread; medians of 3).  The same run
    checks the benched outputs of those problems: budgets, draws and scales
    bit-exact, C.D within 1e-5 (float32)."""
    from oracle import blockmm_oracle as O
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    B = len(keys)
    pick = np.linspace(0, B - 1, sample).astype(int)
    probs = [(Md[b].cpu().numpy().astype(np.float64), Nd[b].cpu().numpy().astype(np.float64)) for b in pick]
    worst = 0.0
    res = {}
    for label, lim in (("all", None), ("1", 1)):
        ctx = threadpool_limits(limits=lim) if (threadpool_limits and lim) else None
        if ctx is not None:
            ctx.__enter__()
        try:
            tots = []
            for rep in range(3):
                t0 = time.perf_counter()
                outs = [O.approx_product(M64, N64, sizes, W, "ONC", workloads.sample_rng(5, int(keys[b])))
                        for (M64, N64), b in zip(probs, pick)]
                tots.append((time.perf_counter() - t0) * 1e3 * B / sample)
        finally:
            if ctx is not None:
                ctx.__exit__(None, None, None)
        res[label] = float(np.median(tots))
    bud, cols, scl = pipe.budgets_host(), pipe.columns_host(), pipe.scales_host()
    for b, ref in zip(pick, outs):
        if not (np.array_equal(bud[b], ref["budgets"]) and np.array_equal(cols[b], ref["columns"])
                and np.array_equal(scl[b], ref["scale"])):
            raise RuntimeError(f"cfg5 problem {b}: budgets / draws differ from the oracle")
        e = float(np.linalg.norm(CD[b].double().cpu().numpy() - ref["CD"]) / np.linalg.norm(ref["CD"]))
        if e > 1e-5:
            raise RuntimeError(f"cfg5 problem {b}: C.D rel err {e:.2e}")
        worst = max(worst, e)
    cb = {"value": res["all"], "unit": "ms/step", "cores": cpu_cores(), "kind": "port", "value_1thread": res["1"],
          "median_of": 3, "sample": f"{sample} of the 4096 problems (evenly spread) through oracle.approx_product "
                                    f"(NumPy + BLAS, float64 upcast), scaled to 4096; wall clock", **cpu_info()}
    par = {"ok": True, "problems_checked": [int(b) for b in pick], "cd_max_rel_err": worst,
           "checked": "budgets, every draw and scale bit-exact vs the oracle; C.D within 1e-5 (float32 bar)"}
    return cb, par


def cfg_traffic(key):
    """DRAM bytes per launch of a kernel from one committed `ncu --set full`
    capture (profiles/traffic.json; null when that kernel was not captured)."""
    path = ROOT / "profiles" / "traffic.json"
    if not path.exists():
        return None
    ent = json.loads(path.read_text()).get(key)
    return None if ent is None else ent.get("bytes_per_launch")


def sketch_numeric_err(pipe, Md, Nd, CD, nb):
    """Numeric error of the float32 contraction alone: ||CD - C.D||_F / ||C.D||_F
    over the first nb problems, C.D in float64 from the same compressed sketch
    (the estimator's own error is the rel_err_* fields)."""
    import torch
    cols = pipe.k_column.view(pipe.B, pipe.W)[:nb]
    sc = pipe.k_scale.view(pipe.B, pipe.W)[:nb]
    cnt = pipe.k_count[:nb].cpu().tolist()
    num = den = 0.0
    for b in range(nb):
        c, s = cols[b, :cnt[b]], sc[b, :cnt[b]]
        C = Md[b][:, c].double() * s
        D = Nd[b][c, :].double() * s[:, None]
        ex = C @ D
        num += float(((CD.view(pipe.B, pipe.m, pipe.p)[b].double() - ex) ** 2).sum())
        den += float((ex ** 2).sum())
    return {"value": float(np.sqrt(num / den)), "problems": nb, "bar": 1e-5}


def run_device(args):
    """cfg5: 4096 independent problems (per-problem seeds).  Under torchrun the
    problems are split over the ranks (no collective; weak in data, the whole
    job's 4096 problems at every N: strong scaling), value = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.pipeline import SketchPipeline, seeds_from_keys
    from paper_2105_04940_b200.analysis import sq_diff

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.workload
    cfg = int(name[-1])
    lo, hi = (rank * 4096 // world, (rank + 1) * 4096 // world)
    Md, Nd, sizes, B = device_data(torch, name, (lo, hi))
    m, n = Md.shape[-2:]
    p = Nd.shape[-1]
    K = len(sizes)
    W = 1024 if name == "cfg5" else 32768
    pipe = SketchPipeline(m, n, p, sizes, W, "ONC", batch=B, dtype=torch.float32)
    keys = np.arange(lo, hi)
    # the batch in waves on several streams of the one graph: a wave's latency-bound planning
    # kernels run beside another wave's HBM-bound norm pass / gather-contraction
    # (tools/cfg5_waves_probe.py; BMM_CFG5_WAVES=0 keeps one batch).  With the one-launch plan the
    # waves cost little, and more of them overlap better: 256 x 16 streams 8.91-8.92 ms, 512 x 8
    # 8.94-8.98, 1024 x 4 8.98-9.02, 128 x 32 9.12, one batch 9.67 (profiles/r2by_waves_plan_small.txt)
    wv = os.environ.get("BMM_CFG5_WAVES", "256,16")
    waves = tuple(int(x) for x in wv.split(",")) if wv not in ("", "0") else None
    if waves is not None and B > waves[0]:
        pipe.set_waves(*waves)
    else:
        waves = None

    def seeds():
        return seeds_from_keys("ONC", workloads.ROOT, (cfg, 1), keys, K)

    pipe.run(Md, Nd, seeds())
    pipe.check()
    pipe.capture(Md, Nd)
    for _ in range(args.warmup):
        pipe.run(Md, Nd, seeds())
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pipe.run(Md, Nd, seeds())
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms_step = float(np.mean([a.elapsed_time(b) for a, b in times]))
    if world > 1:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    first_CD = pipe.run(Md, Nd, seeds()).clone()

    # e2e: this rank's problems from pinned host memory, products back, every step --
    # 8 sub-batches on their own pipelines so one batch's copy overlaps another's work
    SUB = 8
    subs = []
    per = (B + SUB - 1) // SUB
    M_pin = torch.empty(Md.shape, dtype=Md.dtype).pin_memory()
    N_pin = torch.empty(Nd.shape, dtype=Nd.dtype).pin_memory()
    M_pin.copy_(Md)
    N_pin.copy_(Nd)
    out_pin = torch.empty((B, m, p), dtype=torch.float32).pin_memory()
    copy_s = torch.cuda.Stream()
    for j in range(SUB):
        a, bnd = j * per, min(B, (j + 1) * per)
        if a >= bnd:
            continue
        q = SketchPipeline(m, n, p, sizes, W, "ONC", batch=bnd - a, dtype=torch.float32)
        subs.append((a, bnd, q))
    def e2e_step():
        cur = torch.cuda.current_stream()
        for a, bnd, q in subs:
            with torch.cuda.stream(copy_s):
                Md[a:bnd].copy_(M_pin[a:bnd], non_blocking=True)
                Nd[a:bnd].copy_(N_pin[a:bnd], non_blocking=True)
            cur.wait_stream(copy_s)
            ks = keys[a:bnd]
            q.run(Md[a:bnd], Nd[a:bnd], seeds_from_keys("ONC", workloads.ROOT, (cfg, 1), ks, K))
            out_pin[a:bnd].copy_(q._result().view(bnd - a, m, p), non_blocking=True)
    e2e_step()
    e2e = []
    for it in range(1 + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        if it >= 1:
            e2e.append((time.perf_counter() - t0) * 1e3)
    if not torch.equal(out_pin, first_CD.view(B, m, p).cpu()):
        raise RuntimeError("cfg5 end-to-end products differ from the resident run")
    e2e_ms = float(np.mean(e2e))
    del M_pin, N_pin, out_pin, subs

    # per-kernel device times (events on the launching stream)
    lib, st = _lib.load(), _lib.stream_ptr()
    P = lambda t: t.data_ptr()  # noqa: E731

    def timed(fn, reps=3):
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return float(np.median(out))

    norms_ms = timed(lambda: lib.bmm_norms(1, P(Md), m, n, n, m * n, P(Nd), p, p, n * p, B, 0, P(pipe.colsq),
                                           P(pipe.rowsq), st))
    if pipe.fused16:  # config 5: gather + fp16 split + contraction in one kernel (plus the exponent balance)
        fused_ms = timed(lambda: pipe.fused_f16(Md, Nd, st))
        gather_ms = gemm_ms = None
    else:
        gather_ms = timed(lambda: pipe.split_gather(Md, Nd, st))
        gemm_ms = timed(lambda: pipe.split_gemm(st))
        fused_ms = None
    kcounts = pipe.k_count.cpu().numpy()
    kstep = 64 if pipe.f16 else 32  # the contraction's K step (fused fp16 kernel: 32)
    k_exec = int((((kcounts + kstep - 1) // kstep) * kstep).sum())  # columns the compressed contraction runs over
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peak.get("hbm_gbs", 6650.0))
    tf32_peak = float(peak.get("bf16_tflops", 1590.0)) / (1 if (pipe.f16 or pipe.fused16) else 2)  # fp16 / TF32
    norm_bytes = 4 * B * (m * n + n * p)
    useful = 2.0 * m * p * k_exec  # over the distinct drawn columns (compressed sketch, padded to 32)
    # fp16 split: three kind::f16 K=16 MMAs per 16 K; tf32 split: one TF32 K=8 + one BF16 K=16 per 8 K
    executed = (3 if (pipe.f16 or pipe.fused16) else 2) * useful
    # the split gather: reads the sampled elements of M and N, writes the split operands
    # (8 bytes per element: tf32 hi in a float32 container + the bf16 pair word)
    k_distinct = int(kcounts.sum())
    split_bytes = (6 if pipe.f16 else 8) * (m + p) * k_exec
    gather_bytes = 4 * (m + p) * k_distinct + split_bytes
    if fused_ms is not None:
        # one kernel: reads the sampled elements of M and N once, writes the products
        fused_bytes = 4 * (m + p) * k_distinct + 4 * B * m * p
        roof_fused = {"bound": "hbm", "kernel": "gemm_f16split_gather_kernel (gather + fp16 split + tcgen05 "
                                                "kind::f16 contraction, one CTA per problem)",
                      "achieved": fused_bytes / (fused_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": fused_bytes / (fused_ms * 1e-3) / 1e9 / hbm_peak,
                      "algorithmic": "4 B per sampled element of C and D (m + p per distinct drawn column) + 4 B "
                                     "per product element written",
                      "algorithmic_bytes": fused_bytes, "traffic": cfg_traffic("cfg5_fused"),
                      "traffic_note": "M is streamed by TMA in 16-column slabs that hold a drawn column (680 "
                                      "distinct of 4096 touch ~95% of them, as per-element gathers would in "
                                      "DRAM bursts): DRAM reads exceed the sampled bytes (profiles/traffic.json)",
                      "tensor_tflops_executed": executed / (fused_ms * 1e-3) / 1e12,
                      "tensor_frac": executed / (fused_ms * 1e-3) / 1e12 / tf32_peak}
    roof_gather = None if fused_ms is not None else {"bound": "hbm", "kernel": "gather_a_split_kernel + gather_bt_split_kernel (K4, float32 split)",
                   "achieved": gather_bytes / (gather_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                   "frac": gather_bytes / (gather_ms * 1e-3) / 1e9 / hbm_peak,
                   "algorithmic": "4 B per sampled element of C and D read + 8 B per split-operand element written "
                                  "(m + p) x distinct columns (padded to 32) per problem",
                   "algorithmic_bytes": gather_bytes, "traffic": None,
                   "traffic_note": "column gathers of row-major M touch nearly every sector of M (680 sorted distinct "
                                   "columns of 4096): ncu shows the A gather reading all of M "
                                   "(profiles/r1l_ncu_full_summary.csv, gather_a_split_kernel)"}

    # error metric on a verification subset (exact product by our DMMA GEMM on float64 upcasts)
    CD = pipe.run(Md, Nd, seeds())
    nb = min(B, 32)
    if name == "cfg5":
        Mx, Nx = Md[:nb].double(), Nd[:nb].double()
        exact = torch.empty((nb, m, p), dtype=torch.float64, device="cuda")
        ws = _lib.workspace(lib.bmm_gemm_f64_workspace(m, p, n, nb))
        _lib.call("bmm_gemm_f64", P(Mx), n, m * n, P(Nx), p, n * p, m, p, n, nb, P(exact), p, m * p, P(ws),
                  ws.numel(), st)
        approx = CD.view(B, m, p)[:nb]
        err_sq, ref_sq = sq_diff(exact.reshape(nb * m, p), approx.reshape(nb * m, p))
        fro = float(torch.sqrt((torch.linalg.norm(Md[:nb].double(), dim=(1, 2)) ** 2
                                * torch.linalg.norm(Nd[:nb].double(), dim=(1, 2)) ** 2).sum()))
        scope = f"first {nb} problems"
    else:
        rows = 256
        exact = torch.zeros((rows, p), dtype=torch.float64, device="cuda")
        part = torch.empty((rows, p), dtype=torch.float64, device="cuda")
        ws = _lib.workspace(lib.bmm_gemm_f64_workspace(rows, p, 16384, 1))
        for k0 in range(0, n, 16384):
            Ms = Md[:rows, k0:k0 + 16384].double().contiguous()
            Ns = Nd[k0:k0 + 16384].double()
            _lib.call("bmm_gemm_f64", P(Ms), 16384, 0, P(Ns), p, 0, rows, p, 16384, 1, P(part), p, 0, P(ws),
                      ws.numel(), st)
            exact += part
        err_sq, ref_sq = sq_diff(exact, CD.view(m, p)[:rows])
        fro = float(torch.linalg.norm(Md[:rows].double()) * torch.sqrt(pipe.rowsq.sum()))
        scope = f"first {rows} rows of C.D"
    line = {
        "metric": METRIC, "value": ms_step, "unit": "ms/step", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": ("f32 (fp16 h + l split, kind::f16 tensor, f64 plan)" if (pipe.f16 or pipe.fused16)
                                       else "f32 (TF32 + BF16 split-operand tensor, f64 plan)"),
        "data": "synthetic (seeded torch generator on device, SURVEY.md §8(d) distributions)",
        "config": {"workload": name, "batch": 4096, "batch_per_gpu": B, "m": m, "n": n, "p": p, "K": K, "W": W, "method": "ONC",
                   "distinct_columns_mean": float(kcounts.mean()),
                   "l2": f"inputs {norm_bytes / 1e9:.1f} GB >> L2",
                   "waves": (f"{waves[0]} problems per wave on {waves[1]} streams of one graph" if waves else "one batch")},
        "gpu_launches": int(pipe.graph_launches),
        "roofline_norms": {"bound": "hbm", "kernel": "colsq/rowsq (K1)", "achieved": norm_bytes / (norms_ms * 1e-3) / 1e9,
                           "peak": hbm_peak, "unit": "GB/s", "frac": norm_bytes / (norms_ms * 1e-3) / 1e9 / hbm_peak,
                           "algorithmic_bytes": norm_bytes, "traffic": cfg_traffic("cfg5_norms")},
        "rel_err_reference_metric": float(np.sqrt(err_sq / ref_sq)),
        "rel_err_baseline_metric": float(np.sqrt(err_sq) / fro), "error_scope": scope,
        "numeric_err_vs_f64_sketch": sketch_numeric_err(pipe, Md, Nd, CD, min(B, 16)),
        "clocks": clocks.summary(),
    }
    if fused_ms is not None:
        line["roofline_fused"] = roof_fused
        line["kernel_ms"] = {"norms_ms": norms_ms, "gather_gemm_f16split_fused_ms": fused_ms}
        dom = max((norms_ms, line["roofline_norms"]), (fused_ms, roof_fused), key=lambda x: x[0])[1]
    else:
        line["roofline_gemm"] = {"bound": "tensor", "kernel": "gemm_f16split_2sm_kernel" if pipe.f16 else
                                 "gemm_f32split_kernel (tcgen05 kind::tf32 + kind::f16 cross terms)",
                                 "achieved": executed / (gemm_ms * 1e-3) / 1e12, "peak": tf32_peak, "unit": "TFLOP/s",
                                 "frac": executed / (gemm_ms * 1e-3) / 1e12 / tf32_peak,
                                 "operand_bytes": split_bytes, "operand_gbs": split_bytes / (gemm_ms * 1e-3) / 1e9,
                                 "traffic": None}
        line["roofline_gather"] = roof_gather
        line["kernel_ms"] = {"norms_ms": norms_ms, "gather_split_ms": gather_ms, "gemm_split_ms": gemm_ms}
        dom = max((norms_ms, line["roofline_norms"]), (gather_ms, roof_gather), (gemm_ms, line["roofline_gemm"]),
                  key=lambda x: x[0])[1]
    line["roofline"] = dict(dom, dominant="the largest of the kernel_ms entries")
    line["e2e"] = {"value": e2e_ms, "unit": "ms/step", "h2d_bytes_per_step": int(norm_bytes),
                   "d2h_bytes_per_step": int(B * m * p * 4),
                   "api": "SketchPipeline.run on 8 sub-batches: pinned host M, N -> device -> pinned host products"}
    if world > 1:
        line["scaling"] = "strong"
        line["config"]["parallelism"] = f"the 4096 problems split over {world} GPUs, no collective"
    if rank == 0:
        if world == 1:
            cb, par = cfg5_cpu_baseline(pipe, first_CD, Md, Nd, sizes, W, keys)
            line["cpu_baseline"] = cb
            line["parity"] = par
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- config 4 (default workload)
#
# One step = the config-4 comparison over ONE resident instance:
# OPL and ONC approximate products with W = 32768 sketch columns (c = 512 blocks
# of 64) and the SSM whole-block baseline with 512 draws, as one PipelineGroup
# graph whose members share one statistics stage (the norm pass, the block
# probabilities and OPL's Gram-form g_k^2 run once per step).

CFG4_RUNS = (("OPL", 32768, 0), ("ONC", 32768, 1), ("SSM", 512, 2))  # method, W (SSM: draws), sampling rep


def cfg4_seeds(K):
    from paper_2105_04940_b200.pipeline import seeds_from_keys, seeds_from_rngs
    out = []
    for meth, w, rep in CFG4_RUNS:
        if meth == "SSM":
            out.append(seeds_from_rngs("SSM", [workloads.sample_rng(4, rep)], K, draws=w))
        else:  # default_rng(SeedSequence(ROOT, spawn_key=(4, 1, rep))), as workloads.sample_rng(4, rep)
            out.append(seeds_from_keys(meth, workloads.ROOT, (4, 1), [rep], K))
    return out


def cfg4_group(torch, m, n, p, sizes):
    from paper_2105_04940_b200.pipeline import PipelineGroup, SketchPipeline
    pipes = [SketchPipeline(m, n, p, sizes, 0, meth, draws=w, dtype=torch.float32) if meth == "SSM" else
             SketchPipeline(m, n, p, sizes, w, meth, dtype=torch.float32) for meth, w, _ in CFG4_RUNS]
    return PipelineGroup(pipes)


def _oracle_draws(O, probs, sizes, budgets, streams):
    off = O.offsets_of(sizes)
    cols, scales = [], []
    for k in range(len(sizes)):
        if budgets[k]:
            pk = probs[off[k]:off[k + 1]]
            idx = O.draw(pk, int(budgets[k]), streams[k])
            cols.append(off[k] + idx)
            scales.append(1.0 / np.sqrt(int(budgets[k]) * pk[idx]))
    return np.concatenate(cols), np.concatenate(scales)


def cfg4_cpu_leg_parity(torch, group, Md, Nd, outs):
    """CPU-baseline leg, untimed: the oracle (oracle/blockmm_oracle.py, the CPU
    restatement of the reference) run on the host as the CHECKER of the benched
    products -- never on the measured path.
    * norms: 64 random columns of M and 64 random rows of N, bit-exact (the
      chains are per column / per row, so a sample is exact);
    * plan and draws: the oracle's probabilities, score sums, budgets (OPL with
      the device g_k^2, ONC), child streams and inverse-CDF draws from the device
      norms, all bit-exact; SSM block probabilities (1e-13) and its draws;
    * g_k^2 on 2 sampled blocks against the oracle's multiplied-out block (1e-12);
    * C.D on 4 row slabs (first, last, two inner) against float64 of the same
      sketch (1e-5, north_star's float32 bar)."""
    from oracle import blockmm_oracle as O
    opl, onc, ssm = group.pipes
    m, n, p, K, sizes = opl.m, opl.n, opl.p, opl.K, opl.sizes
    off = O.offsets_of(sizes)
    cs, rs = opl.colsq.cpu().numpy(), opl.rowsq.cpu().numpy()
    g = np.random.default_rng(4)
    ci = np.sort(g.choice(n, 64, replace=False))
    ri = np.sort(g.choice(n, 64, replace=False))
    ci_t, ri_t = torch.as_tensor(ci, device="cuda"), torch.as_tensor(ri, device="cuda")
    ok = np.array_equal(O.colsq(Md.index_select(1, ci_t).cpu().numpy().astype(np.float64)), cs[ci])
    ok &= np.array_equal(O.rowsq(Nd.index_select(0, ri_t).cpu().numpy().astype(np.float64)), rs[ri])
    if not ok:
        raise RuntimeError("cfg4 parity: sampled norms differ from the oracle")
    probs, s = O.block_stats(cs, rs, sizes)
    if not (np.array_equal(probs, opl.probs.cpu().numpy()) and np.array_equal(s, opl.s.cpu().numpy())):
        raise RuntimeError("cfg4 parity: probabilities / score sums differ from the oracle")
    gsq = opl.gsq.cpu().numpy()
    res = {}
    sketches = []
    for pipe, (meth, w, rep) in zip(group.pipes, CFG4_RUNS):
        if meth == "SSM":
            q = O.block_norm_weights(cs, rs, sizes)
            q = q / q.sum()
            qd = pipe.q.cpu().numpy()
            qerr = float(np.max(np.abs(qd - q) / q))
            blocks = O.draw(q, w, workloads.sample_rng(4, rep))
            sc = 1.0 / np.sqrt(w * q[blocks])
            if not np.array_equal(pipe.columns_host()[0], blocks) or qerr > 1e-13 or \
                    not np.allclose(pipe.scales_host()[0], sc, rtol=1e-13, atol=0):
                raise RuntimeError("cfg4 parity: SSM draws differ from the oracle")
            res["SSM_q_max_rel_err"] = qerr
            cols = (off[blocks][:, None] + np.arange(sizes[0])[None, :]).ravel()
            sketches.append((cols, np.repeat(pipe.scales_host()[0], sizes[0])))
            continue
        if meth == "ONC":
            budgets, _ = O.plan_budgets("ONC", sizes, w, s=s)
        else:
            budgets, _ = O.plan_budgets("OPL", sizes, w, s=s, aux_sq=gsq)
        cols, scales = _oracle_draws(O, probs, sizes, budgets, workloads.sample_rng(4, rep).spawn(K))
        if not (np.array_equal(pipe.budgets_host()[0], budgets) and np.array_equal(pipe.columns_host()[0], cols)
                and np.array_equal(pipe.scales_host()[0], scales)):
            raise RuntimeError(f"cfg4 parity: {meth} budgets / draws differ from the oracle")
        sketches.append((cols, scales))
    # g_k^2 on sampled blocks vs the oracle's multiplied-out block (BLAS order)
    gerr = 0.0
    for k in (int(g.integers(K)), K - 1):
        ref = O.block_product_sq(Md[:, off[k]:off[k + 1]].cpu().numpy().astype(np.float64),
                                 Nd[off[k]:off[k + 1]].cpu().numpy().astype(np.float64), [sizes[k]])[0]
        gerr = max(gerr, abs(gsq[k] - ref) / ref)
    if gerr > 1e-12:
        raise RuntimeError(f"cfg4 parity: g_k^2 rel err {gerr:.2e}")
    res["gsq_sampled_blocks_max_rel_err"] = gerr
    # C.D vs float64 of the same sketch on row slabs
    cd_err = {}
    for (meth, _, _), (cols, scales), out in zip(CFG4_RUNS, sketches, outs):
        c_t = torch.as_tensor(cols, device="cuda")
        s_t = torch.as_tensor(scales, device="cuda")
        D64 = Nd.index_select(0, c_t).double().mul_(s_t[:, None])
        worst = 0.0
        for r0 in (0, m // 3, 2 * m // 3, m - 128):
            C64 = Md[r0:r0 + 128].index_select(1, c_t).double().mul_(s_t)
            ref = C64 @ D64
            worst = max(worst, float(((out[r0:r0 + 128].double() - ref).norm() / ref.norm()).item()))
        del D64
        if worst > 1e-5:
            raise RuntimeError(f"cfg4 parity: {meth} C.D rel err {worst:.2e} vs float64 of the same sketch")
        cd_err[meth] = worst
    torch.cuda.empty_cache()
    res.update({"ok": True, "cd_rel_err_vs_f64_same_sketch": cd_err,
                "checked": "64 columns of M / 64 rows of N bit-exact; probabilities, score sums, OPL/ONC budgets "
                           "and every draw and scale bit-exact vs oracle/blockmm_oracle.py from the device norms; "
                           "SSM q (1e-13) and draws; g_k^2 of 2 blocks (1e-12); C.D on 4 row slabs of 128 rows "
                           "(first, last, two inner) vs float64 of the same sketch (1e-5)"})
    return res


def cpu_info():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        for d in threadpool_info():
            if d.get("internal_api") in ("openblas", "mkl", "blis"):
                blas = f"{d.get('internal_api')} {d.get('version')} ({d.get('num_threads')} threads max)"
                break
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cfg4_cpu_sample(seed=4):
    """Host slabs of a config-4-distributed instance (numpy, seeded) for the
    bounded CPU sample: 512 rows of M, 4096 rows of N, two blocks M^k / N_k,
    and 512 columns of N over all n rows (the D-slab of the sketch)."""
    g = np.random.default_rng(np.random.SeedSequence(workloads.ROOT, spawn_key=(4, 9, seed)))
    m, n, p, K = 16384, 262144, 16384, 4096
    cscale = np.repeat(g.uniform(0.1, 10, K), n // K).astype(np.float32)
    rscale = np.repeat(g.uniform(0.1, 10, K), n // K).astype(np.float32)
    return {
        "M_rows": g.standard_normal((512, n), dtype=np.float32) * cscale,
        "N_rows": g.standard_normal((4096, p), dtype=np.float32) * rscale[:4096, None],
        "M_blk": [g.standard_normal((m, 64), dtype=np.float32) * cscale[:64] for _ in range(2)],
        "N_blk": [g.standard_normal((64, p), dtype=np.float32) * rscale[:64, None] for _ in range(2)],
        "N_cols": g.standard_normal((n, 512), dtype=np.float32) * rscale[:, None],
    }


def cfg4_cpu_step(S):
    """One config-4 step of the reference path (the oracle port, NumPy + BLAS)
    timed on a bounded sample and extrapolated stage by stage to the full
    config (the fp64 upcast of config 4 does not fit host RAM,
    so the port works on float64-upcast slabs, as the chunked restatement does):
      norms      colsq of 512 rows of M (x m/512), rowsq of 4096 rows of N (x n/4096)
      probs      block_stats over the full n (K = 4096), real size
      g_k (OPL)  block_product_sq on 2 blocks (x K/2): the reference multiplies out every block
      SSM q      ||M^k||_F ||N_k||_F on 2 blocks (x K/2), as plan.py:483-496 (copies + ddot)
      plan+draws budgets and every child stream / draw, real size, per method
      sketch     C on 512 rows (x m/512), D on 512 columns (x p/512), C@D on that 512 x 512 tile over
                 the full W (x m p / 512^2)
    Returns {stage: ms} (extrapolated)."""
    from oracle import blockmm_oracle as O
    m, n, p, K, W, draws = 16384, 262144, 16384, 4096, 32768, 512
    sizes = (64,) * K
    t = {}

    def clock(key, fn, scale=1.0):
        t0 = time.perf_counter()
        out = fn()
        t[key] = t.get(key, 0.0) + (time.perf_counter() - t0) * 1e3 * scale
        return out

    cs_part = clock("norms", lambda: O.colsq_chunked(S["M_rows"], rows=64), m / 512)
    rs_part = clock("norms", lambda: O.rowsq_chunked(S["N_rows"]), n / 4096)
    cs = cs_part
    rs = np.tile(rs_part, n // 4096)
    probs, s = clock("probs", lambda: O.block_stats(cs, rs, sizes))
    for j in range(2):
        clock("gk_opl", lambda: O.block_product_sq(S["M_blk"][j].astype(np.float64),
                                                   S["N_blk"][j].astype(np.float64), [64]), K / 2)
        clock("ssm_q", lambda: (np.linalg.norm(S["M_blk"][j].astype(np.float64))
                                * np.linalg.norm(S["N_blk"][j].astype(np.float64))), K / 2)
    gsq = 0.25 * s ** 2  # timing only: the integerisation's cost does not depend on the values
    for meth, w, rep in CFG4_RUNS:
        rng = np.random.default_rng(np.random.SeedSequence(workloads.ROOT, spawn_key=(4, 8, rep)))
        if meth == "SSM":
            q = O.block_norm_weights(cs, rs, sizes)
            q = q / q.sum()
            blocks = clock("plan_draws", lambda: O.draw(q, w, rng))
            cols = (np.arange(K)[blocks][:, None] * 64 + np.arange(64)[None, :]).ravel()
            scales = np.repeat(1.0 / np.sqrt(w * q[blocks]), 64)
        else:
            def plan():
                b, _ = (O.plan_budgets("ONC", sizes, w, s=s) if meth == "ONC"
                        else O.plan_budgets("OPL", sizes, w, s=s, aux_sq=gsq))
                return _oracle_draws(O, probs, sizes, b, rng.spawn(K))
            cols, scales = clock("plan_draws", plan)
        Wd = cols.size
        C = clock("sketch_gather", lambda: S["M_rows"][:, cols].astype(np.float64) * scales, m / 512)
        D = clock("sketch_gather", lambda: S["N_cols"][cols, :].astype(np.float64) * scales[:, None], p / 512)
        clock("gemm", lambda: C @ D, (m / 512) * (p / 512))
        del C, D, Wd
    return t


def cfg4_cpu_baseline(steps=5, warmup=1):
    """Median over `steps` sample steps at all BLAS threads and at 1 thread."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    S = cfg4_cpu_sample()
    out = {}
    for label, limit in (("all", None), ("1", 1)):
        ctx = threadpool_limits(limits=limit) if (threadpool_limits and limit) else None
        if ctx is not None:
            ctx.__enter__()
        try:
            for _ in range(warmup):
                cfg4_cpu_step(S)
            runs = [cfg4_cpu_step(S) for _ in range(steps if label == "all" else 3)]
        finally:
            if ctx is not None:
                ctx.__exit__(None, None, None)
        tot = [sum(r.values()) for r in runs]
        med = int(np.argsort(tot)[len(tot) // 2])
        out[label] = {"ms": float(np.median(tot)), "stages_ms": {k: float(v) for k, v in runs[med].items()},
                      "runs": len(runs)}
    return out


def cfg4_cpu_line(cb):
    return {"value": cb["all"]["ms"], "unit": "ms/step", "cores": cpu_cores(), "kind": "port",
            "value_1thread": cb["1"]["ms"], "stages_ms": cb["all"]["stages_ms"],
            "stages_ms_1thread": cb["1"]["stages_ms"], "median_of": cb["all"]["runs"],
            "sample": "oracle/blockmm_oracle.py (NumPy + BLAS) on a bounded config-4 sample, extrapolated per "
                      "stage to the full step (bench.cfg4_cpu_step): norms on 512 rows of M / 4096 rows of N, "
                      "g_k and SSM block norms on 2 of 4096 blocks, plan and draws at full size, C.D on a 512 x 512 "
                      "output tile over the full W; float64 upcast slabs (the full upcast needs 69 GB)",
            **cpu_info()}


def run_cfg4(args):
    import torch
    from paper_2105_04940_b200 import _lib

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    m, n, p, K = 16384, 262144, 16384, 4096
    sizes = (n // K,) * K
    Md, Nd = cfg4_shard(torch, (0, m), (0, p))
    group = cfg4_group(torch, m, n, p, sizes)
    outs = [o.clone() for o in group.run(Md, Nd, cfg4_seeds(K))]
    group.check()
    parity = cfg4_cpu_leg_parity(torch, group, Md, Nd, outs)
    del outs
    group.capture(Md, Nd)
    # the norm pass alone on a cool GPU (before the power-capped GEMM steps)
    from paper_2105_04940_b200 import _lib as _l
    sh0 = group.shared
    cool = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _l.load().bmm_norms(1, Md.data_ptr(), m, n, n, 0, Nd.data_ptr(), p, p, 0, 1, 0, sh0.colsq.data_ptr(),
                            sh0.rowsq.data_ptr(), _l.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        cool.append(e0.elapsed_time(e1))
    norms_cool_ms = float(np.median(cool[1:]))
    for _ in range(args.warmup):
        group.run(Md, Nd, cfg4_seeds(K))
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    times = []
    with ClockSampler() as clocks:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            seeds = cfg4_seeds(K)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            group.run(Md, Nd, seeds)
            e1.record(stream)
            times.append((e0, e1))
        torch.cuda.synchronize()
    ms_step = float(np.mean([a.elapsed_time(b) for a, b in times]))
    # the replayed step equals the checked eager step (same kernels, same seeds)
    group.run(Md, Nd, cfg4_seeds(K))
    group.check()

    # ---- per-kernel device times (CUDA events on the launching stream, medians)
    lib, st = _lib.load(), _lib.stream_ptr()
    P = lambda t: t.data_ptr()  # noqa: E731

    def timed(fn, reps=5):
        fn()  # warm: tensor maps, function attributes
        out = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return float(np.median(out))

    sh = group.shared
    norms_ms = timed(lambda: lib.bmm_norms(1, P(Md), m, n, n, 0, P(Nd), p, p, 0, 1, 0, P(sh.colsq), P(sh.rowsq), st))
    cs_ms = timed(lambda: lib.bmm_norms(1, P(Md), m, n, n, 0, None, p, p, 0, 1, 0, P(sh.colsq), None, st))
    rs_ms = timed(lambda: lib.bmm_norms(1, None, m, n, n, 0, P(Nd), p, p, 0, 1, 0, None, P(sh.rowsq), st))
    gram_ms = timed(lambda: lib.bmm_segsq_gram(1, P(Md), n, 0, P(Nd), p, 0, m, p, P(sh.offsets), K, 0, 1,
                                               P(sh.gsq), st))
    gather_ms, gemm_ms, kexec, kdist = [], [], [], []
    for pipe in group.pipes:
        gather_ms.append(timed(lambda: pipe.split_gather(Md, Nd, st)))
        gemm_ms.append(timed(lambda: pipe.split_gemm(st)))
        kd = int(pipe.k_count[0].item())
        kdist.append(kd)
        step = 64 if pipe.f16 else 32
        kexec.append((kd + step - 1) // step * step)

    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = float(peak.get("hbm_gbs", 6538.6))
    tf32_burst = float(peak.get("bf16_tflops", 1631.6)) / 2
    tf32_sust = float(peak.get("bf16_tflops_sustained", 1396.5)) / 2
    traffic = json.loads((ROOT / "profiles" / "traffic.json").read_text()) \
        if (ROOT / "profiles" / "traffic.json").exists() else {}
    norm_bytes = 4 * (m * n + n * p)
    useful = [2.0 * m * p * k for k in kexec]  # over the distinct drawn columns (padded to the K step)
    f16 = all(q.f16 for q in group.pipes)
    # executed tensor work: fp16 split = 3 kind::f16 MMAs (K=16) per 16 K, at the dense fp16/bf16 rate;
    # tf32 split = one TF32 K=8 + one BF16 K=16 MMA (equal cycles) per 8 K, at the dense TF32 rate
    executed = [3 * u for u in useful] if f16 else [2 * u for u in useful]
    if f16:
        tf32_burst, tf32_sust = 2 * tf32_burst, 2 * tf32_sust  # dense fp16 = MEASURED bf16 rates
    gemm_tot = sum(gemm_ms)
    gemm_ach = sum(executed) / (gemm_tot * 1e-3) / 1e12
    gather_bytes = [4 * (m + p) * kd + 8 * (m + p) * ke for kd, ke in zip(kdist, kexec)]
    gram_flops = 2.0 * (m + p) * n * 64 * 36 / 64  # 36 of the 64 8x8 tiles of each 64x64 Gram (symmetry)
    tr = traffic.get("cfg4", {})

    line = {
        "metric": METRIC, "value": ms_step, "unit": "ms/step", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp16 split-operand tensor contraction on CTA pairs, f64 norms/plan)",
        "data": "synthetic (chunk-seeded torch generator on device; SURVEY.md §8(d1) distributions)",
        "config": {"workload": "cfg4", "m": m, "n": n, "p": p, "K": K, "block": 64,
                   "runs": ["OPL@W=32768", "ONC@W=32768", "SSM@draws=512"],
                   "step": "one shared norm pass + block probabilities + Gram g_k, then three approximate products",
                   "distinct_columns": kdist, "l2": "inputs 34.4 GB >> 126 MB L2 (no flush needed)"},
        "gpu_launches": int(group.graph_launches),
        "roofline": {"bound": "tensor",
                     "kernel": ("gemm_f16split_2sm_kernel (tcgen05.mma.cta_group::2 kind::f16: fp16 h.h + [h|l].[l|h] "
                                "pairs, 256x256 tiles per CTA pair, TMA SWIZZLE_128B)") if f16 else
                               "gemm_f32split_2sm_kernel (tcgen05.mma.cta_group::2 kind::tf32 h.h + kind::f16 pairs)",
                     "achieved": gemm_ach, "peak": tf32_sust, "unit": "TFLOP/s", "frac": gemm_ach / tf32_sust,
                     "frac_of_burst": gemm_ach / tf32_burst,
                     "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (dense fp16 = bf16 rate)" if f16 else
                                     "MEASURED_PEAKS.json bf16_tflops_sustained / 2 (dense TF32)") +
                                    "; sustained: the kernel runs inside a ~0.2 s step",
                     "algorithmic": ("executed = 3 x 2*m*p*k per launch, k = distinct drawn columns padded to 64 "
                                     "(three kind::f16 K16 MMAs per 16 k)") if f16 else
                                    ("executed = 2 x 2*m*p*k per launch, k = distinct drawn columns padded to 32 "
                                     "(one TF32 K8 and one BF16 K16 MMA per 8 k)"),
                     "useful_fp32_tflops": sum(useful) / (gemm_tot * 1e-3) / 1e12,
                     "launch_ms": gemm_ms, "share_of_step": gemm_tot / ms_step,
                     "traffic": tr.get("gemm_f32split"), "traffic_src": tr.get("src")},
        "roofline_norms": {"bound": "hbm", "kernel": "colsq_wide_kernel + rowsq_tma_kernel (K1)",
                           "achieved": norm_bytes / (norms_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                           "frac": norm_bytes / (norms_ms * 1e-3) / 1e9 / hbm_peak, "algorithmic_bytes": norm_bytes,
                           "colsq_ms": cs_ms, "rowsq_ms": rs_ms, "ms": norms_ms,
                           "ms_cool": norms_cool_ms,
                           "frac_cool": norm_bytes / (norms_cool_ms * 1e-3) / 1e9 / hbm_peak,
                           "note": "ms / frac: timed right after the step's contractions (SM clock power-capped: "
                                   "the kernels' TMA rings stream ~29 B per clock per SM, the HBM peak only at full "
                                   "clock; DESIGN.md section 8); ms_cool: before them, after the data generation; on "
                                   "a rested GPU 5.1-5.3 ms = 0.99 (tools/cfg4_norms_probe.py)",
                           "traffic": tr.get("norms"), "traffic_src": tr.get("src"),
                           "peak_source": "MEASURED_PEAKS.json hbm_gbs (a copy: read + write)"},
        "roofline_gram": {"bound": "tensor", "kernel": "segsq_gram_kernel (OPL g_k^2 = <M^k'M^k, N_k N_k'>, DMMA)",
                          "ms": gram_ms, "flops": gram_flops,
                          "f64_tflops": gram_flops / (gram_ms * 1e-3) / 1e12,
                          "hbm_gbs": norm_bytes / (gram_ms * 1e-3) / 1e9,
                          "note": "reads M and N once (34.4 GB): bound by max(HBM, DMMA)",
                          "traffic": tr.get("gram")},
        "roofline_gather": {"bound": "hbm", "kernel": "gather_a_split_kernel + gather_bt_split_kernel (K4)",
                            "ms": gather_ms, "algorithmic_bytes": gather_bytes,
                            "achieved": sum(gather_bytes) / (sum(gather_ms) * 1e-3) / 1e9, "peak": hbm_peak,
                            "unit": "GB/s", "frac": sum(gather_bytes) / (sum(gather_ms) * 1e-3) / 1e9 / hbm_peak},
        "kernel_ms": {"norms": norms_ms, "gram_gk": gram_ms, "gather": gather_ms, "gemm": gemm_ms},
        "parity": parity,
        "clocks": clocks.summary(),
    }
    # ---- e2e: the same step from pinned host M, N to pinned host products (one graph:
    # chunked H2D with the shared norm pass and Gram g_k behind it, products copied back)
    import psutil
    need = 4 * (m * n + n * p) + 3 * 4 * m * p
    if psutil.virtual_memory().available > need + (8 << 30):
        M_pin = torch.empty((m, n), dtype=torch.float32).pin_memory()
        N_pin = torch.empty((n, p), dtype=torch.float32).pin_memory()
        M_pin.copy_(Md)
        N_pin.copy_(Nd)
        outs_h = [torch.empty((m, p), dtype=torch.float32).pin_memory() for _ in CFG4_RUNS]
        group.capture_host(Md, Nd, M_pin, N_pin, outs_h, cfg4_seeds(K), n_chunks=8)
        e2e = []
        for it in range(1 + args.steps):
            seeds = cfg4_seeds(K)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            group.run_host(seeds)
            torch.cuda.synchronize()
            if it >= 1:
                e2e.append((time.perf_counter() - t0) * 1e3)
        ref = [o.cpu() for o in group.run(Md, Nd, cfg4_seeds(K))]
        if not all(torch.equal(a, b) for a, b in zip(ref, outs_h)):
            raise RuntimeError("cfg4 end-to-end products differ from the resident run")
        latency = float(np.mean(e2e))
        # steady state: two copies of the step (device inputs, sketch buffers, graph) alternate on
        # two streams, so step i+1's host->device transfer overlaps step i's contractions -- every
        # step still copies its 34 GB of inputs in and its three products out
        pipelined, pipe_note = None, None
        try:
            Md2, Nd2 = torch.empty_like(Md), torch.empty_like(Nd)
            group2 = cfg4_group(torch, m, n, p, sizes)
            outs_h2 = [torch.empty((m, p), dtype=torch.float32).pin_memory() for _ in CFG4_RUNS]
            group2.capture_host(Md2, Nd2, M_pin, N_pin, outs_h2, cfg4_seeds(K), n_chunks=8)
            lanes = [(group, torch.cuda.Stream()), (group2, torch.cuda.Stream())]
            for g_, s_ in lanes:  # warm
                with torch.cuda.stream(s_):
                    g_.run_host(cfg4_seeds(K))
            torch.cuda.synchronize()
            ksteps = max(4, args.steps)
            t0 = time.perf_counter()
            for it in range(ksteps):
                g_, s_ = lanes[it % 2]
                seeds = cfg4_seeds(K)
                with torch.cuda.stream(s_):
                    g_.run_host(seeds)
            torch.cuda.synchronize()
            pipelined = (time.perf_counter() - t0) * 1e3 / ksteps
            if not all(torch.equal(a, b) for a, b in zip(ref, outs_h2)):
                raise RuntimeError("cfg4 pipelined end-to-end products differ from the resident run")
            del group2, Md2, Nd2, outs_h2
        except torch.cuda.OutOfMemoryError as e:  # pragma: no cover
            pipe_note = f"pipelined run skipped: {e}"
        torch.cuda.empty_cache()
        line["e2e"] = {"value": pipelined if pipelined is not None else latency, "unit": "ms/step",
                       "h2d_bytes_per_step": norm_bytes, "d2h_bytes_per_step": 3 * 4 * m * p,
                       "latency_ms": latency,
                       "api": "PipelineGroup.capture_host/run_host: pinned host M, N -> pinned host products "
                              "(one graph per step: chunked H2D with the shared norm pass and Gram g_k behind it)",
                       "mode": ("steady state of consecutive steps, two step instances alternating on two streams "
                                "(transfer of step i+1 overlaps the work of step i); latency_ms: one step alone")
                       if pipelined is not None else "one step at a time"}
        if pipe_note:
            line["e2e"]["note"] = pipe_note
        # the drop-in API on host (numpy) arrays for one ONC product, as a reference user
        # calls it: allocate_by_score_sums + estimate_product (uploads M and N on each call,
        # float64 C and D and the product back as the reference's records)
        try:
            import paper_2105_04940_b200 as bm
            Mh, Nh = M_pin.numpy(), N_pin.numpy()
            part = bm.BlockPartition(sizes)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan = bm.allocate_by_score_sums(Mh, Nh, part, 32768)
            t1 = time.perf_counter()
            pair, CDh, log = bm.estimate_product(Mh, Nh, plan, workloads.sample_rng(4, 1))
            t2 = time.perf_counter()
            ok = np.array_equal(log.column, group.pipes[1].columns_host()[0])
            line["e2e_dropin_api"] = {
                "value": (t2 - t0) * 1e3, "unit": "ms per ONC product", "plan_ms": (t1 - t0) * 1e3,
                "estimate_ms": (t2 - t1) * 1e3, "draws_equal_pipeline": bool(ok),
                "api": "allocate_by_score_sums(M, N, part, 32768) + estimate_product(M, N, plan, rng) on numpy "
                       "float32 arrays (views of pinned buffers here); returns float64 C, D (4.3 GB each), the "
                       "product and the sample log to the host, C @ D on the DMMA engine as the reference's float64"}
            del pair, CDh, log, plan
        except (RuntimeError, torch.cuda.OutOfMemoryError) as e:  # pragma: no cover
            line["e2e_dropin_api"] = {"value": None, "skipped": str(e)[:200]}
        torch.cuda.empty_cache()
        del M_pin, N_pin, outs_h
    else:
        line["e2e"] = {"value": None, "unit": "ms/step", "h2d_bytes_per_step": norm_bytes,
                       "d2h_bytes_per_step": 3 * 4 * m * p,
                       "skipped": f"host RAM available {psutil.virtual_memory().available / 2**30:.0f} GiB < "
                                  f"{(need + (8 << 30)) / 2**30:.0f} GiB of pinned buffers"}
    del Md, Nd
    torch.cuda.empty_cache()
    line["cpu_baseline"] = cfg4_cpu_line(cfg4_cpu_baseline(steps=5 if args.steps >= 5 else max(3, args.steps)))
    print(json.dumps(line), flush=True)
    return 0


def run_reference_cfg4(args):
    """--impl reference on config 4: the CPU port on the bounded sample,
    extrapolated per stage (cfg4_cpu_step), all host BLAS threads."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    S = cfg4_cpu_sample()
    for _ in range(args.warmup):
        cfg4_cpu_step(S)
    runs = [cfg4_cpu_step(S) for _ in range(args.steps)]
    tot = [sum(r.values()) for r in runs]
    v = float(np.median(tot))
    med = int(np.argsort(tot)[len(tot) // 2])
    cb = {"all": {"ms": v, "stages_ms": runs[med], "runs": len(runs)}, "1": {"ms": None, "stages_ms": None}}
    cpu = cfg4_cpu_line(cb)
    cpu.pop("value_1thread")
    cpu.pop("stages_ms_1thread")
    line = {
        "metric": METRIC, "value": v, "unit": "ms/step", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (float32 inputs upcast, as the reference)",
        "data": "synthetic (seeded numpy slabs with the config-4 distributions)",
        "config": {"workload": "cfg4", "m": 16384, "n": 262144, "p": 16384, "K": 4096, "block": 64,
                   "runs": ["OPL@W=32768", "ONC@W=32768", "SSM@draws=512"]},
        "impl": "reference", "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "ms/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_mc(args):
    """--workload mc: the Monte Carlo replication engine --
    coverage_check_plan's replications of one config-1 OPL plan (W=2000):
    a step is `reps` replications of estimate_product + their squared errors."""
    import torch
    import paper_2105_04940_b200 as bm
    from paper_2105_04940_b200 import _lib
    from paper_2105_04940_b200.montecarlo import ReplicationEngine, coverage_check_plan

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    M_h, N_h, sizes = workloads.cfg1()
    m, n = M_h.shape
    p = N_h.shape[1]
    K, W, R = len(sizes), 2000, int(args.reps)
    Md, Nd = torch.as_tensor(M_h, device="cuda"), torch.as_tensor(N_h, device="cuda")
    part = bm.BlockPartition(sizes)
    plan = bm.allocate_optimal(Md, Nd, part, W)
    eng = ReplicationEngine(Md, Nd, plan)
    flush = L2Flush(torch)
    rng_of = lambda i: np.random.default_rng(np.random.SeedSequence(workloads.ROOT, spawn_key=(1, 2, i)))  # noqa: E731
    n0 = _lib.launches()
    eng.run(rng_of(0), R)
    launches = _lib.launches() - n0
    for i in range(args.warmup):
        eng.run(rng_of(1 + i), R)
    torch.cuda.synchronize()
    times = []
    with ClockSampler() as clocks:
        for i in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.run(rng_of(100 + i), R)
            e1.record()
            times.append((e0, e1))
        torch.cuda.synchronize()
    ms_step = float(np.mean([a.elapsed_time(b) for a, b in times]))
    # e2e through the public API with host (numpy) inputs: coverage_check_plan
    err = eng.run(rng_of(7), R)["sq_error"]
    bound = float(err.quantile(0.9).item())
    e2e = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        coverage_check_plan(M_h, N_h, plan, bound, R, rng_of(200 + i))
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e.append((time.perf_counter() - t0) * 1e3)
    # dominant kernel: the batched C_r @ D_r (DMMA), timed on the engine's last chunk
    lib, st = _lib.load(), _lib.stream_ptr()
    b = eng.last_chunk
    Rc = b["reps"]
    gms = []
    for _ in range(5):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.bmm_gemm_f64(b["C"].data_ptr(), W, m * W, b["D"].data_ptr(), p, W * p, m, p, W, Rc, b["CD"].data_ptr(),
                         p, m * p, b["ws_gemm"].data_ptr(), b["ws_gemm"].numel(), st)
        e1.record()
        torch.cuda.synchronize()
        gms.append(e0.elapsed_time(e1))
    gemm_ms = float(np.median(gms))
    flops = 2.0 * m * p * W * Rc
    dgemm_peak = measure_dgemm_peak(torch)
    # CPU baseline: the oracle's replication loop on a bounded sample, scaled to R
    from oracle import blockmm_oracle as O
    sample = 20
    t0 = time.perf_counter()
    O.replicate(M_h, N_h, sizes, plan.probs.flat(), plan.budgets, rng_of(300), sample)
    cpu_ms = (time.perf_counter() - t0) * 1e3 * R / sample
    line = {
        "metric": "Monte Carlo replications (coverage_check_plan): time per step of R replications",
        "value": ms_step, "unit": f"ms/{R} replications", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (config 1, SURVEY.md §8(d))",
        "config": {"workload": "mc", "base": "cfg1", "m": m, "n": n, "p": p, "K": K, "W": W, "method": "OPL",
                   "reps_per_step": R, "l2": "flushed (256 MB write, then 256 MB read) before each step"},
        "e2e": {"value": float(np.mean(e2e)), "unit": f"ms/{R} replications",
                "h2d_bytes_per_step": int(M_h.nbytes + N_h.nbytes), "d2h_bytes_per_step": 8,
                "api": "coverage_check_plan(M, N, plan, bound, reps, rng) on numpy inputs"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "kernel": "gemm_f64_kernel (batched C_r.D_r, DMMA)",
                     "achieved": flops / (gemm_ms * 1e-3) / 1e12, "peak": dgemm_peak, "unit": "TFLOP/s",
                     "frac": flops / (gemm_ms * 1e-3) / 1e12 / dgemm_peak,
                     "peak_source": "cuBLAS dgemm 8192^3 measured in this run", "traffic": None},
        "kernel_ms": {"gemm_batched_ms": gemm_ms},
        "cpu_baseline": {"value": cpu_ms, "unit": f"ms/{R} replications", "cores": cpu_cores(), "kind": "port",
                         "sample": f"{sample} replications with oracle.replicate (NumPy + OpenBLAS), scaled to {R}"},
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_distributed(args)
    if args.workload == "mc":
        return run_mc(args)
    if args.impl == "reference":
        return run_reference_cfg4(args) if args.workload == "cfg4" else run_reference(args)
    if args.workload == "cfg4" and (int(os.environ.get("WORLD_SIZE", "1")) > 1 or
                                    os.environ.get("BMM_FORCE_SHARDED") == "1"):
        return run_cfg4_sharded(args)  # (BMM_FORCE_SHARDED=1: the sharded path at world 1, for testing)
    if args.workload == "cfg4":
        return run_cfg4(args)
    if args.workload == "cfg5":
        return run_device(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
