#!/usr/bin/env python
"""Benchmark of the Frobenius-inversion hot path on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 2 -- one complex n=1024 FP64 matrix,
A = G1 + sqrt(n) I, B = G2, inverted by Frobenius inversion (Alg 1) through
the C ABI (frob_inv, AUTO branch).  One "step" = one full inversion (all SURVEY 8(a) rows
a0-a7).  Inputs (16 MiB) are smaller than L2, so L2 is flushed (256 MiB write) between
timed steps, outside the CUDA-event pairs.

Other workloads (--config): 1 = one n=64 matrix (the line adds a latency table: both branches,
AUTO, complex LU and the batched kernels, warm and cold L2); 3 = batched 65536 x n=32 + 16384 x n=128 (one step = both
sub-batches, sharded across ranks); 4 = matrix sign by Newton, n=2048 (one step = one
full Newton solve, one instance per rank); 5 = one large matrix (--n, default 4096).

Every line also carries: the in-house complex-LU comparator on the same input, the
paper's threshold quantities T_inv, T_mult (Thm 5.1), the roofline of the
GEMM engine, the CPU oracle baseline (rank 0, N=1) and an end-to-end number with host
buffers.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 1|2|3|4|5] [--n N]
Multi-GPU (torchrun): independent problems per rank (instances: seed + rank; batches:
contiguous index shards), no data-path collective, "scaling": "weak"; time = max over ranks.
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
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    return ap.parse_args()


def fp64_alu_peak():
    """Measured FP64 DFMA (non-tensor) peak (tools/fp64_peak.cu)."""
    try:
        with open(PEAKS_FILE) as f:
            d = json.load(f)
        return float(d["dfma_tflops"]), "measured: tools/fp64_peak.cu DFMA register loop, 148 SMs"
    except Exception:
        return 37.2, "nominal: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz"


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
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def torch_empty_pinned_like(torch, t):
    return torch.empty_like(t).pin_memory()


# ------------------------------------------------------------------------------- workloads
class Workload:
    """One config: device-resident step, host-buffer e2e step, units and flops per step."""
    label = ""
    units = 1          # complex inverses per step on this rank
    flops = 0.0        # algorithmic FP64 flops per step on this rank (Frobenius 10 n^3)
    flush = True       # inputs smaller than L2 -> flush between timed steps
    n_ref = 1024       # order used for the comparator / threshold extras
    e2e_mode = "one frob_inv_host call per step (H2D, invert, D2H, synchronise)"

    def step(self):
        raise NotImplementedError

    def e2e_step(self):
        raise NotImplementedError

    def bytes_h2d(self):
        return 0

    def bytes_d2h(self):
        return 0

    def check(self):
        return {}


class SingleMatrix(Workload):
    def __init__(self, fb, torch, dev, n, seed, label):
        import synth
        self.fb, self.torch, self.dev, self.n = fb, torch, dev, n
        self.z_np = synth.config2(n, seed=seed)
        self.z = torch.from_numpy(self.z_np).to(dev)
        self.x = torch.empty_like(self.z)
        self.zh = self.z.cpu().pin_memory()
        self.xh = torch.empty_like(self.zh).pin_memory()
        self.units = 1
        self.flops = 10.0 * n ** 3
        self.flush = 16 * n * n * 2 < 128 * 2 ** 20
        self.n_ref = n
        cfg = 1 if n == 64 else (2 if n == 1024 else 5)
        self.label = (f"config{cfg}: single complex FP64 matrix n={n}, "
                      f"A=G1+sqrt(n)I, B=G2, Frobenius (Alg 1), AUTO branch")

    def step(self):
        self.fb.inv(self.z, out=self.x)

    def e2e_step(self):
        self.fb.inv_host(self.zh, self.xh, device=self.dev)

    def e2e_pipelined(self, k):
        """k steps through frob_inv_host_many (pinned host buffers, the copies of matrices i +- 1
        overlapping inversion i); None when k matrices would not fit a 2 GiB pinned budget."""
        per = 16 * self.n * self.n
        k = min(k, (2 << 30) // per)
        if k < 2:
            return None
        if getattr(self, "_zk", None) is None or self._zk.shape[0] != k:
            self._zk = self.zh.unsqueeze(0).repeat(k, 1, 1).pin_memory()
            self._xk = torch_empty_pinned_like(self.torch, self._zk)
        self.fb.inv_host_many(self._zk, self._xk, device=self.dev)
        return k

    def bytes_h2d(self):
        return self.zh.numel() * 16

    def bytes_d2h(self):
        return self.xh.numel() * 16

    def check(self):
        t = self.torch
        self.fb.inv(self.z, out=self.x)
        r = float(t.linalg.norm(self.z @ self.x - t.eye(self.n, dtype=t.complex128, device=self.dev)))
        return {"residual_fro": r, "residual_bound": 1e-11 * self.n}


class Batched(Workload):
    """Config 3: 65536 x n=32 and 16384 x n=128, shard of this rank."""
    e2e_mode = ("frob_inv_batched_host per part: pinned host buffers, 256 MiB chunks, the copies of "
                "chunks j +- 1 overlapping the inversion of chunk j")

    def __init__(self, fb, torch, dev, rank, world):
        import synth
        from paper_2208_01239_b200 import dist as fdist
        self.fb, self.torch, self.dev = fb, torch, dev
        self.parts = []
        for n, total in ((32, 65536), (128, 16384)):
            b, e = fdist.shard_range(total, rank, world)
            z = torch.from_numpy(synth.batch(n, e - b, seed=0, start=b)).to(dev)
            self.parts.append((n, z, torch.empty_like(z)))
        self.units = sum(p[1].shape[0] for p in self.parts)
        self.flops = sum(10.0 * p[0] ** 3 * p[1].shape[0] for p in self.parts)
        self.flush = False
        self.n_ref = 128
        self.host = [(p[1].cpu().pin_memory(), torch.empty_like(p[1], device="cpu").pin_memory()) for p in self.parts]
        self.label = "config3: 65536 x n=32 + 16384 x n=128 complex FP64 (shift 8, seed+index), batched Frobenius, AUTO"

    def step(self):
        for n, z, x in self.parts:
            self.fb.inv_batched(z, out=x)

    def e2e_step(self):
        # the host-buffer entry point, pipelined in 256 MiB chunks (copies overlap the inversions)
        for (n, z, x), (zh, xh) in zip(self.parts, self.host):
            self.fb.inv_batched_host(zh, xh, device=self.dev)

    def bytes_h2d(self):
        return sum(h[0].numel() * 16 for h in self.host)

    def bytes_d2h(self):
        return self.bytes_h2d()

    def check(self):
        t = self.torch
        out = {}
        for n, z, x in self.parts:
            _, info, bu = self.fb.inv_batched(z, out=x)
            e = t.matmul(z[:512], x[:512]) - t.eye(n, dtype=t.complex128, device=self.dev)
            out[f"n{n}"] = {"singular": int((info != 0).sum()), "branch_b": int((bu == 2).sum()),
                            "residual_fro_max_first512": float(t.linalg.norm(e, dim=(1, 2)).max())}
        return out


class SignNewton(Workload):
    """Config 4: sign(Z) by Newton, n=2048, one instance per rank."""
    e2e_mode = "per step: H2D of Z, frob_sign_newton, D2H of S"

    def __init__(self, fb, torch, dev, n, seed):
        import synth
        self.fb, self.torch, self.dev, self.n = fb, torch, dev, n
        z, s, lam, sinv = synth.sign_instance(n, seed=seed)
        self.ref = torch.from_numpy((s * np.sign(lam.real)[None, :]) @ sinv).to(dev)
        self.z = torch.from_numpy(z).to(dev)
        self.zh = self.z.cpu().pin_memory()
        self.sh = torch.empty_like(self.zh).pin_memory()
        _, it, _ = fb.sign(self.z, tol=1e-12, max_iter=50)
        self.iters = it
        self.units = it             # complex inversions per Newton solve
        self.flops = 10.0 * n ** 3 * it
        self.flush = False
        self.n_ref = n
        self.label = f"config4: matrix sign by Newton, complex FP64 n={n}, tol 1e-12 (Frobenius inversions)"

    def step(self):
        self.fb.sign(self.z, tol=1e-12, max_iter=50)

    def e2e_step(self):
        z = self.zh.to(self.dev, non_blocking=True)
        s, _, _ = self.fb.sign(z, tol=1e-12, max_iter=50)
        self.sh.copy_(s)

    def bytes_h2d(self):
        return self.zh.numel() * 16

    def bytes_d2h(self):
        return self.sh.numel() * 16

    def check(self):
        s, it, d = self.fb.sign(self.z, tol=1e-12, max_iter=50)
        t = self.torch
        rel = float(t.linalg.norm(s - self.ref) / t.linalg.norm(self.ref))
        return {"newton_iters": it, "final_delta": d, "rel_err_vs_closed_form": rel}


# ------------------------------------------------------------------------------- reference arm
def run_reference(args, rank):
    """The CPU oracle as the reference arm (tier rule): same metric, config and unit."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    if args.config in (1, 2, 5):
        n = args.n or {1: 64, 2: 1024, 5: 4096}[args.config]
        z = synth.config2(n, seed=0)
        work = lambda: oracle.frob_inv(z)  # noqa: E731
        units, label = 1, f"config{args.config}: single complex FP64 matrix n={n}, Frobenius (Alg 1)"
        sample = f"{args.steps} oracle frob_inv calls at n={n}"
    elif args.config == 3:
        z32 = synth.batch(32, 2048, seed=0)
        z128 = synth.batch(128, 16, seed=0)

        def work():
            for m in z32:
                oracle.frob_inv(m)
            for m in z128:
                oracle.frob_inv(m)
        units, label = 2048 + 16, "config3 sample: 2048 x n=32 + 16 x n=128 (same generator), Frobenius"
        sample = "per step: 2048 n=32 + 16 n=128 matrices of the config-3 set (bounded sample)"
    else:
        z, _, _, _ = synth.sign_instance(512, seed=0)
        work = lambda: oracle.sign_newton(z, tol=1e-12, max_iter=50)  # noqa: E731
        units, label = 13, "config4 sample: sign Newton at n=512 (same generator)"
        sample = "per step: one Newton sign solve at n=512 (bounded sample of config 4)"
    for _ in range(min(args.warmup, 1)):
        work()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        work()
    dt = time.perf_counter() - t0
    v = units * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generators)", "config": {"workload": label, "l2": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, wl):
    """Oracle on the box's host cores, bounded sample (~10 s), same unit."""
    import oracle
    import synth
    oracle.build()
    t0 = time.perf_counter()
    cnt = 0
    if isinstance(wl, SingleMatrix):
        while True:
            oracle.frob_inv(wl.z_np)
            cnt += 1
            if time.perf_counter() - t0 > 10.0 or cnt >= 20:
                break
        sample = f"{cnt} oracle frob_inv calls (plain C, OpenMP) on the same n={wl.n} input"
        dt_all = time.perf_counter() - t0
        # the complex Gauss-Jordan oracle timed separately, and one thread at n <= 1024
        extra = {}
        t1, c1 = time.perf_counter(), 0
        while True:
            oracle.zinv_gj(wl.z_np)
            c1 += 1
            if time.perf_counter() - t1 > 5.0 or c1 >= 20:
                break
        extra["zinv_gj_oracle_per_s"] = c1 / (time.perf_counter() - t1)
        if wl.n <= 1024:
            nt = oracle.num_threads()
            oracle.set_threads(1)
            t1, c1 = time.perf_counter(), 0
            while True:
                oracle.frob_inv(wl.z_np)
                c1 += 1
                if time.perf_counter() - t1 > 5.0 or c1 >= 5:
                    break
            extra["frob_oracle_1thread_per_s"] = c1 / (time.perf_counter() - t1)
            oracle.set_threads(nt)
        return {"value": cnt / dt_all, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                "sample": sample, **extra}
    elif isinstance(wl, Batched):
        zs = synth.batch(32, 4096, seed=0)
        for m in zs:
            oracle.frob_inv(m)
            cnt += 1
            if time.perf_counter() - t0 > 8.0:
                break
        sample = f"{cnt} n=32 matrices of the config-3 set (oracle frob_inv); n=128 omitted"
    else:
        z, _, _, _ = synth.sign_instance(512, seed=0)
        _, it, _ = oracle.sign_newton(z, tol=1e-12, max_iter=50)
        cnt = it
        sample = f"one Newton sign solve at n=512 ({it} oracle Frobenius inversions; n=2048 too slow)"
    dt = time.perf_counter() - t0
    return {"value": cnt / dt, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle", "sample": sample}


# ------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    from paper_2208_01239_b200 import dist as fdist
    ws, rank, local = fdist.env()
    if args.impl == "reference":
        return run_reference(args, rank)

    import torch
    import torch.distributed as dist

    import paper_2208_01239_b200 as fb
    from paper_2208_01239_b200 import frobinv as fbi

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    fbi.load()

    if args.config in (1, 2, 5):
        wl = SingleMatrix(fb, torch, dev, args.n or {1: 64, 2: 1024, 5: 4096}[args.config],
                          fdist.instance_seed(0, rank), "")
    elif args.config == 3:
        wl = Batched(fb, torch, dev, rank, ws)
    else:
        wl = SignNewton(fb, torch, dev, args.n or 2048, fdist.instance_seed(0, rank))

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def timed(fn, steps, warmup, flush_l2):
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
        wl.step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = fbi.launch_count()
    with ClockSampler(local) as clk:
        times = timed(wl.step, args.steps, 0, wl.flush)
    launches = fbi.launch_count() - l0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = fdist.max_over_ranks(sum(times), dev)
    units_all = fdist.sum_over_ranks(wl.units, dev)
    ms_step = total_ms / args.steps
    value = units_all * args.steps / (total_ms / 1e3)
    flops_all = fdist.sum_over_ranks(wl.flops, dev)
    peak, peak_src = fp64_peak()

    extras = {}
    if not args.no_extras:
        n = wl.n_ref
        import synth
        zr = torch.from_numpy(synth.config2(n, seed=rank)).to(dev)
        xr = torch.empty_like(zr)
        t_zinv = statistics.median(timed(lambda: fb.zinv(zr, out=xr), 5, 2, True))
        t_frob = statistics.median(timed(lambda: fb.inv(zr, out=xr), 5, 2, True))
        a = zr.real.contiguous()
        ainv = torch.empty_like(a)
        cm = torch.empty_like(a)
        t_inv = statistics.median(timed(lambda: fb.dinv(a, out=ainv), 5, 2, True))
        t_mult = statistics.median(timed(lambda: fb.dgemm(a, ainv, cm), 5, 2, True))
        ratio = t_inv / t_mult
        r_z = t_zinv / t_inv
        lam = 1.0
        if n <= 64:
            # BASELINE config 1: latency of both branches, AUTO, complex LU and the
            # batched kernels on one matrix; median of 100 after 10 warm-ups, warm and cold L2
            lat = {}
            zb = zr[None].contiguous()
            cases = {"frob_auto": lambda: fb.inv(zr, out=xr), "frob_branch_a": lambda: fb.inv(zr, out=xr, branch="a"),
                     "frob_branch_b": lambda: fb.inv(zr, out=xr, branch="b"), "zinv_lu": lambda: fb.zinv(zr, out=xr),
                     "frob_batched_kernel": lambda: fb.inv_batched(zb), "zinv_batched_kernel": lambda: fb.zinv_batched(zb)}
            for nm_, f_ in cases.items():
                lat[nm_] = {"warm_l2_us": 1e3 * statistics.median(timed(f_, 100, 10, False)),
                            "cold_l2_us": 1e3 * statistics.median(timed(f_, 100, 10, True))}
            extras["latency_config1"] = lat
        extras["comparison_single_n"] = {
            "n": n, "frobenius_ms": t_frob, "zinv_lu_ms": t_zinv,
            "frobenius_tflops_alg": 10.0 * n ** 3 / t_frob / 1e9, "zinv_lu_tflops_alg": 8.0 * n ** 3 / t_zinv / 1e9,
            "frob_over_zinv_time": t_frob / t_zinv}
        extras["threshold"] = {
            "n": n, "T_inv_ms": t_inv, "T_mult_ms": t_mult, "ratio_Tinv_Tmult": ratio,
            "paper_threshold_lambda_half": 1.25, "paper_threshold_lambda_one": 1.5, "lambda": lam, "r_z": r_z,
            "break_even_general": (2 + lam) / (r_z - 2) if r_z > 2 else None,
            "predicted_frob_faster": bool(r_z > 2 and ratio > (2 + lam) / (r_z - 2)),
            "measured_frob_faster": bool(t_frob < t_zinv)}
        if isinstance(wl, Batched):
            # batched Frobenius vs the batched complex Gauss-Jordan comparator (n <= 64): the
            # config-3 n = 32 shard, and n = 64 from the same generator (crossover evidence)
            cmp = {}
            z64 = torch.from_numpy(synth.batch(64, 16384, seed=0)).to(dev)
            # (n = 128: the complex comparator needs a 2-CTA cluster per matrix -- a complex 128 x 128
            # matrix fits neither one SM's registers nor its shared memory; the real ones do)
            for nn, zz in ((32, wl.parts[0][1]), (64, z64), (128, wl.parts[1][1])):
                tb_f = statistics.median(timed(lambda: fb.inv_batched(zz), 3, 1, False))
                tb_z = statistics.median(timed(lambda: fb.zinv_batched(zz), 3, 1, False))
                cnt = int(zz.shape[0])
                cmp[f"n{nn}"] = {"count": cnt, "frob_ms": tb_f, "zinv_lu_ms": tb_z, "frob_over_zinv_time": tb_f / tb_z,
                                 "frob_inverses_per_s": cnt / tb_f * 1e3, "zinv_inverses_per_s": cnt / tb_z * 1e3,
                                 "frob_tflops_alg": 10.0 * nn ** 3 * cnt / tb_f / 1e9,
                                 "zinv_tflops_alg": 8.0 * nn ** 3 * cnt / tb_z / 1e9}
            extras["batched_comparison"] = cmp
        # NEXT-1 (fused first step) and Alg 5 (randomized) on the same input
        t_fused = statistics.median(timed(lambda: fb.inv(zr, out=xr, fused=True), 5, 2, True))
        t_rand = statistics.median(timed(lambda: fb.inv_rand(zr, mu=0.5, out=xr), 5, 2, True))
        extras["comparison_single_n"].update({
            "frobenius_fused_first_step_ms": t_fused, "frobenius_fused_tflops_alg": (28.0 / 3.0) * n ** 3 / t_fused / 1e9,
            "frobenius_randomized_ms": t_rand})
        # NEXT-4: HPD inversion, Cholesky-based Frobenius variant (Alg 6) vs complex Cholesky (Alg 8)
        zh = torch.from_numpy(synth.hpd(n, seed=rank)).to(dev)
        t_h6 = statistics.median(timed(lambda: fb.hpd_inv(zh, out=xr, check=False), 5, 2, True))
        t_h8 = statistics.median(timed(lambda: fb.zhpd_inv(zh, out=xr, check=False), 5, 2, True))
        extras["hpd_comparison"] = {"n": n, "frob_hpd_alg6_ms": t_h6, "complex_cholesky_alg8_ms": t_h8,
                                    "alg6_over_alg8_time": t_h6 / t_h8}
        # GEMM engine (DMMA) at the n x n x n shape of the three Frobenius GEMMs
        ach = 2.0 * n ** 3 / t_mult / 1e9
        extras["roofline_gemm"] = {"bound": "tensor", "kernel": "gemm_kernel<double> (DMMA m8n8k4), n x n x n",
                                   "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                                   "peak_source": peak_src}
        # dominant kernel of the timed step: a separate instrumented pass (CUDA events recorded by
        # the library on the stream each kernel is launched on), never inside the timed region
        fbi.profile_enable(True)
        pw = timed(wl.step, max(2, min(args.steps, 5)), 1, wl.flush)
        prof = fbi.profile_read()
        fbi.profile_enable(False)
        if prof:
            name, d = max(prof.items(), key=lambda kv: kv[1]["total_ms"])
            avg_ms = d["total_ms"] / max(1, d["launches"])
            ach_k = d["flops"] / max(1, d["launches"]) / (avg_ms * 1e-3) / 1e12
            # DMMA kernels: the GEMM engine and lu2's trailing updates (NEXT / BULK)
            tensor = name.startswith("gemm") or name.startswith("lu_update2") or name.startswith("lu_next2")
            pk, pk_src = (peak, peak_src) if tensor else fp64_alu_peak()
            steps_prof = len(pw) + 1
            traffic = None
            try:  # DRAM bytes per launch from this round's committed ncu --set full capture
                # (captured at n = 1024, the config 2 default, and at n = 4096 under "<name> n=4096")
                with open(os.path.join(ROOT, "profiles", "r01", "dram_traffic.json")) as f:
                    tab = json.load(f)
                wn = getattr(wl, "n", None)
                tr = tab.get(name) if wn == 1024 else tab.get(f"{name} n={wn}")
                if tr and "batched" not in name:
                    traffic = tr["bytes_per_launch"]
            except Exception:
                pass
            extras["roofline"] = {
                "bound": "tensor" if tensor else "alu", "kernel": name, "achieved": ach_k, "peak": pk,
                "unit": "TFLOP/s", "frac": ach_k / pk, "traffic": traffic, "peak_source": pk_src,
                "flops_per_launch": d["flops"] / max(1, d["launches"]), "avg_launch_ms": avg_ms,
                "launches_per_step": d["launches"] / steps_prof,
                "share_of_step": d["total_ms"] / steps_prof / statistics.median(pw),
                "note": ("FP64 pipe; the LU panel is a latency-bound pivot chain (one pivot search + "
                         "rank-1 update per column), so its fraction of the FP64 peak is small by nature; "
                         "its launch duration includes the programmatic-dependent-launch wait for its "
                         "predecessor (kernels overlap by design), so share_of_step can exceed the "
                         "critical-path share"
                         if not tensor else "DMMA tensor pipe")}
            extras["kernel_profile"] = {k: {"launches_per_step": v["launches"] / steps_prof,
                                            "ms_per_step": v["total_ms"] / steps_prof,
                                            "tflops": v["flops"] / (v["total_ms"] * 1e-3) / 1e12 if v["total_ms"] else None}
                                        for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])}
        e2e = timed(wl.e2e_step, max(3, args.steps // 2), 1, False)
        e2e_ms = fdist.max_over_ranks(statistics.median(e2e), dev)
        extras["e2e"] = {"value": units_all * 1e3 / e2e_ms, "unit": UNIT,
                         "h2d_bytes_per_step": int(wl.bytes_h2d()), "d2h_bytes_per_step": int(wl.bytes_d2h()),
                         "mode": wl.e2e_mode}
        if hasattr(wl, "e2e_pipelined"):
            # the streaming entry point: K steps per call, each step's own H2D and D2H inside the
            # timed region, overlapped with the neighbouring steps' inversions
            kk = max(4, args.steps)
            got = wl.e2e_pipelined(kk)  # warm-up (and pinned buffers)
            if got:
                reps = []
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    wl.e2e_pipelined(kk)
                    e1.record(stream)
                    torch.cuda.synchronize()
                    reps.append(e0.elapsed_time(e1) / got)
                pm = fdist.max_over_ranks(statistics.median(reps), dev)
                single = extras["e2e"]
                extras["e2e"] = {"value": units_all * 1e3 / pm, "unit": UNIT,
                                 "h2d_bytes_per_step": int(wl.bytes_h2d()), "d2h_bytes_per_step": int(wl.bytes_d2h()),
                                 "mode": f"frob_inv_host_many over {got} steps per call: the host->device copy of "
                                         f"step i+1 and the device->host copy of step i-1 overlap step i's inversion",
                                 "single_call": {"value": single["value"], "mode": single["mode"]}}
                if wl.flush:
                    extras["e2e"]["l2"] = ("not flushed between the steps of one pipelined call (the "
                                           "device-resident value flushes L2 before every step)")
    chk = wl.check()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, wl)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE generators, seed = rank / index)",
            "config": {"workload": wl.label, "l2": ("flushed (256 MiB write) between timed steps" if wl.flush
                                                    else "inputs larger than L2 / not flushed"),
                       "parallelism": f"{ws} rank(s), independent problems"},
            "tflops_alg": flops_all / (total_ms / args.steps * 1e-3) / 1e12,
            "step_roofline_frac": flops_all / (total_ms / args.steps * 1e-3) / 1e12 / (peak * ws),
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk.summary(),
            "check": chk,
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
