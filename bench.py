#!/usr/bin/env python
"""Benchmark: fmaps/s of the batched regularized functional-map solver on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2] [--gather] [--no-cpu-baseline]

One "step" = one pass of the hot path over one batch (BASELINE cfg2: 64 shape
pairs, k=200, d=256, n=5000): device-resident G, R, M -> C through the C ABI
(`fmap_solve_f32_dev`: validation + solver kernel), the region the reference
times (bench.hpp:136-140: assembly + factorization + solve; generation, mask
and Gram excluded).  `e2e` is the same metric through the host-buffer C ABI
(`fmap_solve_f32`) with pinned host G, R, M in and C out every step.
`pipeline` adds the device end-to-end path (Phi, Mass, F, ev -> C).

Multi-GPU (torchrun, one process per GPU): pairs are sharded, each rank owns
a fixed 64-pair slice (weak scaling), no collective in the timed region; the
device time is the max over ranks.  `--gather` also times the final gather of
C to rank 0 (NCCL), reported separately.

`--impl reference` times the CPU reference path (the C++ restatement of the
reference's batched route, oracle/, with every host thread) on a bounded
sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fmaps/sec at k=200 (batch 64) 1/2/4/8 B200; % FP32 peak; vs CPU ref"
UNIT = "fmaps/s"
PAPER_2080TI_FMAPS = 1000.0 / 7.05  # PAPER.md:278, batch 1, RTX 2080 Ti (context only)


def flops_per_fmap(k: int) -> float:
    """north_star convention: k^4/3 + k^3 flops per fmap."""
    return k ** 4 / 3.0 + k ** 3


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.lines: list[str] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.15)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload --
def make_inputs(workload: str, rank: int, device):
    """Generate the rank's shard on the host (seeded), project + Gram + mask on
    the GPU with our own kernels (untimed, like the reference's build_problems)."""
    import torch
    from paper_2604_10377_b200 import synth, fmsolve, _lib
    import ctypes as C
    cfg = synth.CONFIGS[workload]
    b = cfg.batch
    data = synth.make_batch(cfg, q0=rank * b, count=b)
    t = {k: torch.from_numpy(v).to(device) for k, v in data.items()}
    k, d = cfg.k, cfg.d
    A = torch.empty((b, k, d), device=device)
    B = torch.empty((b, k, d), device=device)
    G = torch.empty((b, k, k), device=device)
    R = torch.empty((b, k, k), device=device)
    M = torch.empty((b, k, k), device=device)
    ctx = _lib.context(device.index or 0)
    ctx.set_stream(torch.cuda.current_stream(device).cuda_stream)
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    L = ctx._lib
    h = ctx.handle
    for st in (L.fmap_project_f32_dev(h, b, cfg.n_src, k, d, P(t["phi1"]), P(t["mass1"]), P(t["F1"]), P(A)),
               L.fmap_project_f32_dev(h, b, cfg.n_tgt, k, d, P(t["phi2"]), P(t["mass2"]), P(t["F2"]), P(B)),
               L.fmap_normal_equations_f32_dev(h, b, k, d, P(A), P(B), P(G), P(R)),
               L.fmap_mask_f32_dev(h, b, k, P(t["ev1"]), P(t["ev2"]), 1, cfg.sigma, P(M))):
        if st != 0:
            raise RuntimeError(ctx.last_error())
    torch.cuda.synchronize(device)
    ctx.set_stream(None)
    return cfg, t, G, R, M


# ----------------------------------------------------------------- our arm --
def run_ours(args):
    import torch
    import torch.distributed as dist
    import ctypes as C
    from paper_2604_10377_b200 import fmsolve, _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)

    cfg, t, G, R, M = make_inputs(args.workload, rank, device)
    b, k = cfg.batch, cfg.k
    C_out = torch.empty_like(G)
    opts = fmsolve.SolverOptions(compute_residual=False).to_c()
    ctx = _lib.context(local)
    stream = torch.cuda.Stream(device)
    ctx.set_stream(stream.cuda_stream)
    L, h = ctx._lib, ctx.handle
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)  # > L2 (126 MB)

    def step():
        rep = _lib.ReportC()
        st = L.fmap_solve_f32_dev(h, b, k, P(G), P(R), P(M), cfg.lam, C.byref(opts), P(C_out), C.byref(rep))
        if st != 0:
            raise RuntimeError(f"solve failed: {ctx.last_error()}")
        return rep

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step()
    launches_per_step = ctx.last_launch_count
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()

    total_ms, kernel_ms = 0.0, []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(device)
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()                      # L2 flush, outside the timed events
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            rep = step()                           # the API call syncs its stream at the end
            with torch.cuda.stream(stream):
                e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            kernel_ms.append(rep.wall_seconds * 1e3)
        torch.cuda.synchronize(device)
    if world > 1:
        tt = torch.tensor([total_ms], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())

    fmaps = world * b * args.steps
    value = fmaps / (total_ms * 1e-3)
    ms_per_step = total_ms / args.steps

    gather_ms = None
    if world > 1 and args.gather:
        out = torch.empty((world,) + tuple(C_out.shape), device=device) if True else None
        torch.cuda.synchronize(device)
        dist.barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record()
        dist.all_gather_into_tensor(out, C_out)
        g1.record()
        g1.synchronize()
        gt = torch.tensor([g0.elapsed_time(g1)], device=device, dtype=torch.float64)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather_ms = float(gt.item())

    result = None
    if rank == 0:
        kavg = statistics.mean(kernel_ms)
        flops = b * flops_per_fmap(k)
        sms = torch.cuda.get_device_properties(device).multi_processor_count
        clocks = clk.summary()
        peak_max = sms * 128 * 2 * 1965e6 / 1e12   # FP32 SIMT at clocks.max.sm
        achieved = flops / (kavg * 1e-3) / 1e12
        traffic = _ncu_traffic()
        bf16_peak = _measured_bf16_peak()
        roofline = {
            # compute-bound kernel: the trailing updates run on tcgen05 (3xTF32), the
            # panel chain on the FP32 pipe; the north_star's denominator is FP32 peak
            "bound": "tensor",
            "achieved": round(achieved, 3), "peak": round(peak_max, 3), "unit": "TFLOP/s",
            "frac": round(achieved / peak_max, 4), "traffic": traffic,
            "kernel": "chol_tc_kernel", "kernel_ms": round(kavg, 4),
            "flops_per_launch": flops,
            "peak_note": ("achieved counts the north_star's k^4/3 + k^3 flops per fmap; peak = FP32 "
                          "SIMT (north_star's denominator) derived as SMs x 128 lanes x 2 x 1965 MHz "
                          "(MEASURED_PEAKS.json has no FP32 figure); frac_at_sampled_clock uses the "
                          "median SM clock sampled during the timed region"),
        }
        if bf16_peak:
            roofline["frac_of_measured_bf16_tensor"] = round(achieved / bf16_peak, 5)
        if clocks.get("sm_mhz"):
            roofline["frac_at_sampled_clock"] = round(
                achieved / (sms * 128 * 2 * clocks["sm_mhz"] * 1e6 / 1e12), 4)
        result = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic: seeded BASELINE cfg generator (mass-orthonormal Phi via QR, "
                    "N(0,1) features, U(0,1)j^2 spectra to 200), random-init, no dataset",
            "config": {"workload": args.workload, "pairs_per_gpu": b, "global_batch": b * world,
                       "k": k, "d": cfg.d, "n": cfg.n_src, "lambda": cfg.lam,
                       "mask": f"resolvent sigma={cfg.sigma}", "parallelism": f"pairs sharded x{world}",
                       "l2": "flushed between steps (256 MiB write outside the timed events)",
                       "timed": "solve-only, device-resident G,R,M -> C via fmap_solve_f32_dev "
                                "(validation + tcgen05/TMEM Cholesky solver), the reference's timed region"},
            "roofline": roofline,
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clocks,
            "vs_paper_2080ti_batch1": round(value / PAPER_2080TI_FMAPS, 1),
        }
        if gather_ms is not None:
            result["gather_ms"] = round(gather_ms, 4)
    # e2e + pipeline: each rank measures its own, max over ranks
    e2e_ms = _e2e(args, cfg, G, R, M, device, ctx, stream)
    pipe_ms = _pipeline(args, cfg, t, device, stream)
    if world > 1:
        tt = torch.tensor([e2e_ms, pipe_ms], device=device, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, pipe_ms = (float(x) for x in tt.tolist())
    if rank == 0:
        nbytes = b * k * k * 4
        result["e2e"] = {"value": round(world * b / (e2e_ms * 1e-3), 2), "unit": UNIT,
                         "h2d_bytes_per_step": 3 * nbytes, "d2h_bytes_per_step": nbytes,
                         "ms_per_step": round(e2e_ms, 4),
                         "api": "fmap_solve_f32 (host G,R,M pinned -> C): 8 pair chunks, H2D / validation+solve / D2H overlapped on 2 copy + 2 compute streams, device validation incl."}
        result["pipeline"] = {"value": round(world * b / (pipe_ms * 1e-3), 2), "unit": UNIT,
                              "ms_per_step": round(pipe_ms, 4),
                              "api": "fmap_pipeline_f32_dev: Phi,Mass,F,ev -> projection, Gram/RHS, "
                                     "fused resolvent mask, solver (device-resident)"}
        if not args.no_cpu_baseline and world == 1:
            result["cpu_baseline"] = _cpu_baseline(args, G, R, M, k, cfg.lam)
        print(json.dumps(result), flush=True)
    ctx.set_stream(None)
    if world > 1:
        dist.destroy_process_group()


def _measured_bf16_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
    except Exception:
        return None


def _ncu_traffic():
    """dram bytes per launch of the solver from the committed ncu --set full summary."""
    for p in sorted((ROOT / "profiles").glob("ncu_solver_*.json"), reverse=True):
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            continue
    return None


def _e2e(args, cfg, G, R, M, device, ctx, stream) -> float:
    """Same metric through the host C ABI with pinned buffers, copies included."""
    import torch
    import ctypes as C
    from paper_2604_10377_b200 import fmsolve, _lib
    b, k = cfg.batch, cfg.k
    hG, hR, hM = (x.cpu().pin_memory() for x in (G, R, M))
    hC = torch.empty_like(hG).pin_memory()
    opts = fmsolve.SolverOptions(compute_residual=False).to_c()
    P = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    L, h = ctx._lib, ctx.handle

    def call():
        rep = _lib.ReportC()
        st = L.fmap_solve_f32(h, b, k, P(hG), P(hR), P(hM), cfg.lam, C.byref(opts), P(hC), C.byref(rep))
        if st != 0:
            raise RuntimeError(ctx.last_error())
    for _ in range(max(1, args.warmup)):
        call()
    steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(steps):
        call()                      # returns after C is back in pinned host memory
    return (time.perf_counter() - t0) * 1e3 / steps


def _pipeline(args, cfg, t, device, stream) -> float:
    import torch
    from paper_2604_10377_b200 import fmsolve
    opts = fmsolve.SolverOptions(compute_residual=False)
    run = lambda: fmsolve.pipeline_device(  # noqa: E731
        t["phi1"], t["mass1"], t["F1"], t["ev1"], t["phi2"], t["mass2"], t["F2"], t["ev2"],
        lam=cfg.lam, sigma=cfg.sigma, bidirectional=cfg.bidirectional, opts=opts)
    for _ in range(max(1, args.warmup)):
        run()
    steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / steps


def _cpu_baseline(args, G, R, M, k, lam) -> dict:
    """Oracle (restated reference batched route, all host threads) on a bounded
    sample of the same inputs; plus the serial rowwise route on a smaller one."""
    import oracle
    threads = os.cpu_count() or 1
    pairs = int(os.environ.get("FMAP_CPU_SAMPLE_PAIRS", "16"))
    g, r, m = (x[:pairs].cpu().numpy() for x in (G, R, M))
    res = oracle.solve(g, r, m, lam, route="batched", dtype=np.float32, threads=threads)
    val = pairs / res.wall_seconds
    g1, r1, m1 = g[:1], r[:1], m[:1]
    ser = oracle.solve(g1, r1, m1, lam, route="rowwise", dtype=np.float32)
    return {"value": round(val, 3), "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{pairs} cfg2 pairs (k={k}) through the restated reference batched route "
                      f"(partial-pivot LU + rcond, std::thread x{threads}), f32, same inputs",
            "serial_rowwise": {"value": round(1 / ser.wall_seconds, 3), "unit": UNIT, "cores": 1,
                               "sample": "1 cfg2 pair, rowwise route (solver.hpp:174-218)"}}


# ----------------------------------------------------------- reference arm --
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle
    from paper_2604_10377_b200 import synth
    cfg = synth.CONFIGS[args.workload]
    pairs = int(os.environ.get("FMAP_REF_SAMPLE_PAIRS", "8"))
    threads = os.cpu_count() or 1
    # inputs: the same generator; G, R in float64 on the host, cast like the device path
    data = synth.make_batch(cfg, 0, pairs)
    G, R, M = [], [], []
    for q in range(pairs):
        pair = {kk: v[q] for kk, v in data.items()}
        A, B = synth.descriptors_f64(pair)
        G.append(A @ A.T)
        R.append(B @ A.T)
        M.append(oracle.mask(1, pair["ev1"].astype(np.float64), pair["ev2"].astype(np.float64), cfg.sigma))
    G, R, M = (np.stack(x).astype(np.float32) for x in (G, R, M))
    times = []
    for i in range(args.warmup + args.steps):
        res = oracle.solve(G, R, M, cfg.lam, route="batched", dtype=np.float32, threads=threads)
        if i >= args.warmup:
            times.append(res.wall_seconds)
    total = sum(times)
    value = pairs * len(times) / total
    out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total / len(times), 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
           "impl": "reference",
           "data": "synthetic: seeded BASELINE cfg generator, bounded sample",
           "config": {"workload": args.workload, "sample_pairs_per_step": pairs, "k": cfg.k, "d": cfg.d,
                      "n": cfg.n_src, "lambda": cfg.lam, "mask": f"resolvent sigma={cfg.sigma}",
                      "timed": "reference batched route (solver.hpp:220-322 restated, oracle/), "
                               "assembly + LU + rcond + solve; residual excluded"},
           "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
                            "sample": f"{pairs} pairs per step, std::thread x{threads}"},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--gather", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
