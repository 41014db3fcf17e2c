#!/usr/bin/env python
"""Benchmark of the Frobenius-inversion hot path on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 2 -- one complex n=1024 FP64 matrix,
A = G1 + sqrt(n) I, B = G2, inverted by Frobenius inversion (Alg 1) through
the C ABI (frob_inv, AUTO branch).  One "step" = one full inversion (all SURVEY 8(a)
rows a0-a7).  Inputs (16 MiB) are smaller than L2, so L2 is flushed (256 MiB write)
between timed steps, outside the CUDA-event pairs.

Also reported on the same line: the in-house complex-LU comparator (zinv_lu) on the
same input, the paper's threshold quantities T_inv, T_mult (Thm 5.1), the
roofline of the dominant kernel, the CPU oracle baseline and an end-to-end number with
host buffers.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 2|5] [--n N]
Multi-GPU (torchrun): every rank inverts its own instance (seed + rank): independent
problems, no data-path collective, "scaling": "weak"; timing = max over ranks.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "complex_inverses_per_sec"
UNIT = "inverses/s"
PEAKS_FILE = os.path.join(ROOT, "profiles", "fp64_peak.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[2, 5])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def fp64_peak():
    """Measured FP64 tensor (DMMA) peak on this pool's B200 (tools/fp64_peak.cu)."""
    try:
        with open(PEAKS_FILE) as f:
            d = json.load(f)
        return float(d["dmma_tflops"]), "measured: tools/fp64_peak.cu DMMA m8n8k4 register loop, 148 SMs"
    except Exception:
        return 37.2, "nominal: 148 SMs x 128 FP64 flop/clk x 1.965 GHz"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------------------------- reference arm
def run_reference(args, n, ws, rank):
    """The CPU oracle as the reference arm (tier rule): same metric, config and unit."""
    if rank != 0:
        return
    import oracle
    import synth
    z = synth.config2(n, seed=0)
    for _ in range(min(args.warmup, 1)):
        oracle.frob_inv(z)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.frob_inv(z)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config 2 generator, seed 0)",
        "config": {"workload": f"config{args.config}: single complex FP64 matrix n={n}, Frobenius (Alg 1)",
                   "n": n, "l2": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"{args.steps} oracle frob_inv calls at n={n}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    ws, rank, local = dist_env()
    n = args.n or (1024 if args.config == 2 else 4096)
    if args.impl == "reference":
        return run_reference(args, n, ws, rank)

    import torch
    import torch.distributed as dist

    import paper_2208_01239_b200 as fb
    from paper_2208_01239_b200 import frobinv as fbi
    import synth

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = fbi.load()

    z_np = synth.config2(n, seed=rank)           # instance per rank (weak scaling)
    z = torch.from_numpy(z_np).to(dev)
    x = torch.empty_like(z)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step_frob():
        fb.inv(z, out=x)

    def step_zinv():
        fb.zinv(z, out=x)

    def timed(fn, steps, warmup, flush_l2=True):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for e0, e1 in evs:
            if flush_l2:
                flush.zero_()
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        return [e0.elapsed_time(e1) for e0, e1 in evs]

    # ---------------------------------------------------------------- main timed region
    for _ in range(args.warmup):
        step_frob()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = fbi.launch_count()
    with ClockSampler(local) as clk:
        times = timed(step_frob, args.steps, 0)
    launches = fbi.launch_count() - l0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(times)
    if ws > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    value = ws * args.steps / (total_ms / 1e3)
    flops = 10.0 * n ** 3  # Frobenius literal: 2 T_inv + 3 T_mult = 10 n^3
    peak, peak_src = fp64_peak()

    extras = {}
    if not args.no_extras:
        # comparator and threshold quantities (Thm 5.1) on the same GPU, same input
        zt = timed(step_zinv, max(5, args.steps // 2), 2)
        t_zinv = statistics.median(zt)
        a = z.real.contiguous()
        ainv = torch.empty_like(a)
        cm = torch.empty_like(a)
        t_inv = statistics.median(timed(lambda: fb.dinv(a, out=ainv), 10, 2))
        t_mult = statistics.median(timed(lambda: fb.dgemm(a, ainv, cm), 10, 2))
        t_frob_med = statistics.median(times)
        ratio = t_inv / t_mult
        r_z = t_zinv / t_inv
        lam = 1.0
        pred = ratio > (2 + lam) / (r_z - 2) if r_z > 2 else False
        extras = {
            "frobenius": {"ms_median": t_frob_med, "tflops_alg": flops / t_frob_med / 1e9},
            "zinv_lu": {"ms_median": t_zinv, "inverses_per_sec": 1e3 / t_zinv,
                        "tflops_alg": 8.0 * n ** 3 / t_zinv / 1e9},
            "threshold": {"T_inv_ms": t_inv, "T_mult_ms": t_mult, "ratio_Tinv_Tmult": ratio,
                          "paper_threshold_lambda_half": 1.25, "paper_threshold_lambda_one": 1.5,
                          "lambda": lam, "r_z": r_z, "break_even_general": (2 + lam) / (r_z - 2) if r_z > 2 else None,
                          "predicted_frob_faster": bool(pred), "measured_frob_faster": bool(t_frob_med < t_zinv)},
            "gemm_tflops_nnn": 2.0 * n ** 3 / t_mult / 1e9,
        }
        # roofline of the dominant kernel: the DMMA GEMM engine at the n x n x n shape the
        # three Frobenius GEMMs use (same kernel, same stream, CUDA events, L2 flushed)
        extras["roofline"] = {
            "bound": "tensor", "kernel": "gemm_kernel<double> (DMMA m8n8k4)",
            "achieved": 2.0 * n ** 3 / t_mult / 1e9, "peak": peak, "unit": "TFLOP/s",
            "frac": (2.0 * n ** 3 / t_mult / 1e9) / peak, "traffic": None,
            "peak_source": peak_src,
        }
        # end-to-end through the C ABI with pinned host buffers (H2D + compute + D2H)
        zh = z.cpu().pin_memory()
        xh = torch.empty_like(zh).pin_memory()
        e2e_t = timed(lambda: fb.inv_host(zh, xh, device=dev), max(3, args.steps // 2), 1)
        extras["e2e"] = {"value": ws * 1e3 / statistics.median(e2e_t), "unit": UNIT,
                         "h2d_bytes_per_step": int(zh.numel() * 16), "d2h_bytes_per_step": int(xh.numel() * 16)}

    # correctness spot check of the timed output (residual, independent torch GEMM)
    fb.inv(z, out=x)
    res = float(torch.linalg.norm(z @ x - torch.eye(n, dtype=torch.complex128, device=dev)))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        t0 = time.perf_counter()
        cnt = 0
        while True:
            oracle.frob_inv(z_np)
            cnt += 1
            if time.perf_counter() - t0 > 10.0 or cnt >= 20:
                break
        dt = time.perf_counter() - t0
        cpu = {"value": cnt / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
               "sample": f"{cnt} oracle frob_inv calls (plain C, OpenMP) on the same n={n} input"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE config 2 generator, seed = rank)",
            "config": {"workload": f"config{args.config}: single complex FP64 matrix n={n}, Frobenius (Alg 1), AUTO branch",
                       "n": n, "l2": "flushed (256 MiB write) between timed steps", "parallelism": f"replicas x{ws}"},
            "tflops_alg": flops / (ms_step * 1e-3) / 1e12,
            "step_roofline_frac": flops / (ms_step * 1e-3) / 1e12 / peak,
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk.summary(),
            "residual_fro": res,
        }
        line.update(extras)
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
