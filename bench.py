#!/usr/bin/env python
"""Benchmark of the Frobenius-inversion hot path on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 5 at its headline size -- one complex FP64 matrix of
order n = 16384 (A = G1 + sqrt(n) I, B = G2, seed + rank; A and B are 2 GiB each), the largest
single-GPU configuration, inverted by Frobenius inversion (Alg 1) through the C ABI
(frob_inv, AUTO branch).  One "step" = one full inversion (every SURVEY 8(a) row a0-a7) per rank.
Inputs (4 GiB) exceed L2 (126 MB), so no flush is needed between steps.

The line also carries: the in-house complex-LU comparator on the same input (the paper's
`X\\eye(n)`), the paper's threshold quantities at n (T_inv, T_mult and the measured
lambda of Thm 5.1), NEXT-1 / Alg 5 timings, the HPD comparison with T_pinv / T_mult
against Thm 6.2's 7/6 (capped at n = 4096), the roofline of the dominant kernel (CUDA events on its
launch stream, an instrumented pass after the timed region), sketch parity against the committed
oracle fixture, an end-to-end number through the host-buffer C-ABI call, and the CPU oracle
baseline (n^3-scaled from a bounded sample: the plain oracle cannot invert n = 16384 in minutes).

Other workloads (--config): 1 = one n=64 matrix (+ latency table); 2 = one n=1024 matrix;
3 = batched 65536 x n=32 + 16384 x n=128 (one step = both sub-batches, sharded across ranks);
4 = matrix sign by Newton, n=2048 (one step = one full Newton solve); 5 = one large matrix
(--n, default 16384).  --instances K (configs 4/5): K independent instances spread over the ranks
(K/N per rank, "scaling": "strong"; default: one per rank, "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 1|2|3|4|5] [--n N] [--instances K]
Multi-GPU (torchrun): independent problems per rank (instances seed + global index; batches:
contiguous index shards), no data-path collective; time = max over ranks; per-rank records
all-gathered (paper_2208_01239_b200.dist.summarize).
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
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r02", "dram_traffic.json")
SKETCH_META = os.path.join(ROOT, "tests", "golden", "sketch_config5.json")
DEFAULT_N = {1: 64, 2: 1024, 5: 16384}
ORACLE_SAMPLE_N = 2048     # config 5: the oracle's bounded sample (n^3-scaled to the workload's n)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--instances", type=int, default=None,
                    help="configs 4/5: total independent instances over all ranks (strong scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    return ap.parse_args()


def _peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f)
    except Exception:
        return {}


def fp64_alu_peak():
    """Measured FP64 DFMA (non-tensor) peak (tools/fp64_peak.cu)."""
    d = _peaks()
    if "dfma_tflops" in d:
        return float(d["dfma_tflops"]), "measured: tools/fp64_peak.cu DFMA register loop, 148 SMs"
    return 37.2, "nominal: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz"


def fp64_peak():
    """Measured FP64 tensor (DMMA) peak on this pool's B200 (tools/fp64_peak.cu)."""
    d = _peaks()
    if "dmma_tflops" in d:
        return float(d["dmma_tflops"]), "measured: tools/fp64_peak.cu DMMA m8n8k4 register loop, 148 SMs"
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


# ------------------------------------------------------------------------------- workloads
def single_label(n):
    cfg = 1 if n == 64 else (2 if n == 1024 else 5)
    return (f"config{cfg}: single complex FP64 matrix n={n}, A=G1+sqrt(n)I, B=G2 (seed + instance), "
            f"Frobenius inversion (Alg 1), AUTO branch")


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

    def stats(self):
        return {}


class SingleMatrix(Workload):
    """Configs 1, 2, 5: `instances` independent matrices per rank (global index -> seed)."""

    def __init__(self, fb, torch, dev, n, seeds):
        import synth
        self.fb, self.torch, self.dev, self.n = fb, torch, dev, n
        self.seeds = list(seeds)
        self.z_np0 = synth.config2(n, seed=self.seeds[0])
        self.zs = [torch.from_numpy(self.z_np0).to(dev)] + \
                  [torch.from_numpy(synth.config2(n, seed=s)).to(dev) for s in self.seeds[1:]]
        self.z = self.zs[0]
        self.xs = [torch.empty_like(z) for z in self.zs]
        self.x = self.xs[0]
        self.zh = self.z.cpu().pin_memory()
        self.xh = torch.empty_like(self.zh).pin_memory()
        self.units = len(self.zs)
        self.flops = 10.0 * n ** 3 * self.units
        self.flush = 16 * n * n * 2 < 128 * 2 ** 20
        self.n_ref = n
        self.label = single_label(n)
        self.branch_counts = {}

    def step(self):
        for z, x in zip(self.zs, self.xs):
            self.fb.inv(z, out=x)

    def e2e_step(self):
        self.fb.inv_host(self.zh, self.xh, device=self.dev)

    def e2e_pipelined(self, k):
        """k steps through frob_inv_host_many (pinned host buffers, the copies of matrices i +- 1
        overlapping inversion i; k DISTINCT matrices, seeds 1000 + i); None when fewer than two
        matrices (inputs and outputs) fit a 24 GiB pinned budget."""
        import synth
        per = 16 * self.n * self.n
        k = min(k, (24 << 30) // (2 * per))
        if k < 2:
            return None
        if getattr(self, "_zk", None) is None or self._zk.shape[0] != k:
            self._zk = self.torch.stack([self.torch.from_numpy(synth.config2(self.n, seed=1000 + i))
                                         for i in range(k)]).pin_memory()
            self._xk = self.torch.empty_like(self._zk).pin_memory()
        self.fb.inv_host_many(self._zk, self._xk, device=self.dev)
        return k

    def bytes_h2d(self):
        return self.zh.numel() * 16

    def bytes_d2h(self):
        return self.xh.numel() * 16

    def check(self):
        t, n = self.torch, self.n
        out = {}
        x, info = self.fb.inv(self.z, out=self.x, info=True)
        out["branch_used"] = info["branch_used"]
        out["rho_a"] = info["rho_a"]
        # per-column residuals ||Z x_j - e_j|| in fp64 on the host (8 sampled columns)
        rng = np.random.default_rng(n)
        cols = rng.choice(n, size=min(8, n), replace=False)
        xs = x[:, t.from_numpy(cols).to(self.dev)].cpu().numpy()
        worst = 0.0
        for k, j in enumerate(cols):
            r = self.z_np0 @ xs[:, k]
            r[j] -= 1.0
            worst = max(worst, float(np.linalg.norm(r)))
        out["column_residual_max"] = worst
        kappa = None
        try:
            with open(SKETCH_META) as f:
                meta = json.load(f).get(str(n))
        except Exception:
            meta = None
        if meta and self.seeds[0] == 0:
            # sketch parity against the committed oracle fixture (tests/golden/make_sketch.py)
            import synth
            yo = t.from_numpy(np.load(os.path.join(ROOT, "tests", "golden", meta["file"]))).to(self.dev)
            r = t.from_numpy(synth.rademacher(n, meta["k"], seed=0)).to(self.dev).to(t.complex128)
            rel = float(t.linalg.norm(x @ r - yo) / t.linalg.norm(yo))
            kappa = meta["kappa2_est"]
            kf = max(1.0, kappa / 1e4)
            out["parity_vs_oracle"] = {"sketch_rel_fro": rel, "bound": 1e-10 * kf, "kappa2_est": kappa,
                                       "method": "||(X_gpu - X_oracle) R||_F / ||X_oracle R||_F, R = +-1 (n x 64); "
                                                 "X_oracle R committed by tests/golden/make_sketch.py",
                                       "ok": rel <= 1e-10 * kf}
        kf = max(1.0, (kappa or 1.0) / 1e4)
        out["column_residual_bound"] = 1e-11 * math.sqrt(n) * kf
        if n <= 8192:
            res = float(t.linalg.norm(self.z @ x - t.eye(n, dtype=t.complex128, device=self.dev)))
            out["residual_fro"] = res
            out["residual_bound"] = 1e-11 * n * kf
        return out

    def stats(self):
        return {"instances": self.units, "seeds": self.seeds}


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

    def stats(self):
        c = self.check()
        return {"matrices": self.units, "branch_b": {k: v["branch_b"] for k, v in c.items()},
                "singular": {k: v["singular"] for k, v in c.items()}}


class SignNewton(Workload):
    """Config 4: sign(Z) by Newton, n=2048, `instances` per rank."""
    e2e_mode = "per step: H2D of Z, frob_sign_newton, D2H of S"

    def __init__(self, fb, torch, dev, n, seeds):
        import synth
        self.fb, self.torch, self.dev, self.n = fb, torch, dev, n
        self.seeds = list(seeds)
        self.zs, self.refs = [], []
        for sd in self.seeds:
            z, s, lam, sinv = synth.sign_instance(n, seed=sd)
            self.refs.append(torch.from_numpy((s * np.sign(lam.real)[None, :]) @ sinv).to(dev))
            self.zs.append(torch.from_numpy(z).to(dev))
        self.z = self.zs[0]
        self.zh = self.z.cpu().pin_memory()
        self.sh = torch.empty_like(self.zh).pin_memory()
        self.iters = []
        for z in self.zs:
            _, it, _ = fb.sign(z, tol=1e-12, max_iter=50)
            self.iters.append(it)
        self.units = sum(self.iters)   # complex inversions per step
        self.flops = 10.0 * n ** 3 * self.units
        self.flush = False
        self.n_ref = n
        self.label = f"config4: matrix sign by Newton, complex FP64 n={n}, tol 1e-12 (Frobenius inversions)"

    def step(self):
        for z in self.zs:
            self.fb.sign(z, tol=1e-12, max_iter=50)

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
        rel = float(t.linalg.norm(s - self.refs[0]) / t.linalg.norm(self.refs[0]))
        return {"newton_iters": it, "final_delta": d, "rel_err_vs_closed_form": rel}

    def stats(self):
        return {"instances": len(self.zs), "newton_iters": self.iters, "seeds": self.seeds}


# ------------------------------------------------------------------------------- oracle legs
def _oracle_threads():
    import oracle
    return oracle.num_threads()


def oracle_sample(config, n_work):
    """(work(), units per call, scale, label, sample) of the bounded oracle sample for a config.
    scale converts the sample's inverses/s into the workload's unit (config 5: (n_s / n)^3)."""
    import oracle
    import synth
    oracle.build()
    if config in (1, 2):
        z = synth.config2(n_work, seed=0)
        return (lambda: oracle.frob_inv(z)), 1, 1.0, f"oracle frob_inv (plain C, OpenMP) at n={n_work}"
    if config == 5:
        ns = min(n_work, ORACLE_SAMPLE_N)
        z = synth.config2(ns, seed=0)
        return ((lambda: oracle.frob_inv(z)), 1, (ns / n_work) ** 3,
                f"oracle frob_inv (plain C, OpenMP) at n={ns} (config-5 generator), rate scaled by (n_s/n)^3 = "
                f"({ns}/{n_work})^3 to inverses/s at n={n_work}: the plain oracle cannot invert n={n_work} "
                f"within the run (an upper bound of its rate there: larger n only loses cache locality)")
    if config == 3:
        z32 = synth.batch(32, 2048, seed=0)
        z128 = synth.batch(128, 16, seed=0)

        def work():
            oracle.frob_inv_many(z32)
            oracle.frob_inv_many(z128)
        return work, 2048 + 16, 1.0, "per call: 2048 n=32 + 16 n=128 matrices of the config-3 set (oracle frob_inv_many)"
    z, _, _, _ = synth.sign_instance(512, seed=0)
    return ((lambda: oracle.sign_newton(z, tol=1e-12, max_iter=50)), 13, 1.0,
            "per call: one Newton sign solve at n=512 (13 oracle Frobenius inversions; n=2048 too slow)")


def run_reference(args, rank, ws, n_work, label):
    """The CPU oracle as the reference arm (tier rule): same metric, config label and unit; rank 0."""
    if rank != 0:
        return
    work, units, scale, sample = oracle_sample(args.config, n_work)
    for _ in range(min(args.warmup, 1)):
        work()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        work()
    dt = time.perf_counter() - t0
    v = units * args.steps / dt * scale
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE generators)", "config": {"workload": label, "l2": "cpu"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": _oracle_threads(), "kind": "oracle",
                         "sample": f"each step: {sample}"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, n_work):
    """Oracle on the box's host cores, bounded sample (~10-20 s), in the workload's unit."""
    work, units, scale, sample = oracle_sample(args.config, n_work)
    t0 = time.perf_counter()
    cnt = 0
    while True:
        work()
        cnt += 1
        if time.perf_counter() - t0 > 12.0 or cnt >= 20:
            break
    dt = time.perf_counter() - t0
    out = {"value": units * cnt / dt * scale, "unit": UNIT, "cores": _oracle_threads(), "kind": "oracle",
           "sample": f"{cnt} calls: {sample}", "sample_seconds": dt}
    if args.config in (1, 2, 5):
        import oracle
        import synth
        ns = min(n_work, ORACLE_SAMPLE_N)
        z = synth.config2(ns, seed=0)
        t1 = time.perf_counter()
        oracle.zinv_gj(z)
        out["zinv_gj_oracle_seconds_at_n_sample"] = time.perf_counter() - t1
    return out


# ------------------------------------------------------------------------------- our arm
def main():
    args = parse()
    from paper_2208_01239_b200 import dist as fdist
    ws, rank, local = fdist.env()
    n_work = args.n or DEFAULT_N.get(args.config, 2048)
    if args.config == 3:
        label = Batched.label if hasattr(Batched, "label") and Batched.label else \
            "config3: 65536 x n=32 + 16384 x n=128 complex FP64 (shift 8, seed+index), batched Frobenius, AUTO"
    elif args.config == 4:
        label = f"config4: matrix sign by Newton, complex FP64 n={args.n or 2048}, tol 1e-12 (Frobenius inversions)"
    else:
        label = single_label(n_work)
    if args.impl == "reference":
        return run_reference(args, rank, ws, n_work, label)

    import torch
    import torch.distributed as dist

    import paper_2208_01239_b200 as fb
    from paper_2208_01239_b200 import frobinv as fbi

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
        print(f"[bench rank {rank}] process group: backend={dist.get_backend()} world_size={dist.get_world_size()}",
              file=sys.stderr, flush=True)
    fbi.load()

    strong = args.instances is not None and args.config in (4, 5, 1, 2)
    if strong:
        inst = fdist.instances_for_rank(args.instances, rank, ws)
    else:
        inst = [rank]
    seeds = [fdist.instance_seed(0, g) for g in inst]
    if args.config in (1, 2, 5):
        wl = SingleMatrix(fb, torch, dev, n_work, seeds)
    elif args.config == 3:
        wl = Batched(fb, torch, dev, rank, ws)
    else:
        wl = SignNewton(fb, torch, dev, args.n or 2048, seeds)

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
    summ = fdist.summarize(times, wl.units, {"rank": rank, **wl.stats()}, dev)
    total_ms, units_all, ms_step, value = summ["total_ms"], summ["units_all"], summ["ms_per_step"], summ["value"]
    flops_all = fdist.sum_over_ranks(wl.flops, dev)
    peak, peak_src = fp64_peak()

    extras = {}
    if not args.no_extras:
        extras.update(run_extras(args, wl, fb, fbi, torch, dev, rank, timed, peak, peak_src, units_all, stream,
                                 fdist))
    chk = wl.check()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, n_work)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE generators, seed = global instance / index)",
            "config": {"workload": wl.label,
                       "l2": ("flushed (256 MiB write) between timed steps" if wl.flush
                              else "inputs larger than L2 / not flushed"),
                       "parallelism": f"{ws} rank(s), independent problems, {wl.units} unit(s) per rank per step",
                       "instances_total": args.instances if strong else ws},
            "tflops_alg": flops_all / (total_ms / args.steps * 1e-3) / 1e12,
            "step_roofline_frac": flops_all / (total_ms / args.steps * 1e-3) / 1e12 / (peak * ws),
            "gpu_launches": int(launches),
            "gpu_launches_per_step": launches / args.steps,
            "clocks": clk.summary(),
            "check": chk,
            "per_rank": summ["per_rank"],
        }
        if ws > 1:
            line["comm"] = {"backend": "nccl", "world_size": ws,
                            "data_path_collectives": 0, "note": "barrier + max/sum reductions + all_gather of per-rank records"}
        line.update(extras)
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def _kernel_groups(prof):
    """Profiler entries -> kernels: role scopes ("step:*", brackets around many kernels) are dropped,
    and the three Frobenius GEMMs (one gemm_kernel<double> launch each, n x n x n) form one kernel."""
    out = {}
    for k, v in prof.items():
        if k.startswith("step:"):
            continue
        key = "gemm_kernel<double> Frobenius GEMMs a3/a4/a6 (n x n x n)" if k.startswith("gemm:frob_") else k
        d = out.setdefault(key, {"launches": 0, "total_ms": 0.0, "flops": 0.0, "parts": []})
        d["launches"] += v["launches"]
        d["total_ms"] += v["total_ms"]
        d["flops"] += v["flops"]
        d["parts"].append(k)
    return out


def _traffic_for(kernel, n):
    """DRAM bytes per launch from this round's committed ncu --set full capture of the SAME kernel at
    the SAME shape (profiles/r02/dram_traffic.json); None when no such capture exists."""
    try:
        with open(TRAFFIC_FILE) as f:
            tab = json.load(f)
    except Exception:
        return None, None
    rec = tab.get(f"{kernel} n={n}")
    if not rec:
        return None, None
    return rec.get("bytes_per_launch"), rec.get("source")


def run_extras(args, wl, fb, fbi, torch, dev, rank, timed, peak, peak_src, units_all, stream, fdist):
    import synth
    extras = {}
    n = wl.n_ref
    big = n > 4096
    reps, warm = (3, 1) if big else (5, 2)
    zr = wl.z if isinstance(wl, (SingleMatrix, SignNewton)) else torch.from_numpy(synth.config2(n, seed=rank)).to(dev)
    xr = torch.empty_like(zr)
    t_zinv = statistics.median(timed(lambda: fb.zinv(zr, out=xr), reps, warm, not big))
    t_frob = statistics.median(timed(lambda: fb.inv(zr, out=xr), reps, warm, not big))
    a = zr.real.contiguous()
    ainv = torch.empty_like(a)
    cm = torch.empty_like(a)
    t_inv = statistics.median(timed(lambda: fb.dinv(a, out=ainv), reps, warm, not big))
    t_mult = statistics.median(timed(lambda: fb.dgemm(a, ainv, cm), reps, warm, not big))
    # lambda (Thm 5.1): a triangular x dense product on the same engine, relative to T_mult
    low = torch.tril(a)
    t_trmm = statistics.median(timed(lambda: fb.dtrmm(low, ainv, uplo="lower", c=cm), reps, warm, not big))
    del low
    lam = t_trmm / t_mult
    t_fused = statistics.median(timed(lambda: fb.inv(zr, out=xr, fused=True), reps, warm, not big))
    ratio = t_inv / t_mult
    r_z = t_zinv / t_inv
    if n <= 64:
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
        "n": n, "frobenius_ms": t_frob, "zinv_lu_ms": t_zinv, "frobenius_fused_first_step_ms": t_fused,
        "frobenius_tflops_alg": 10.0 * n ** 3 / t_frob / 1e9, "zinv_lu_tflops_alg": 8.0 * n ** 3 / t_zinv / 1e9,
        "frobenius_fused_tflops_alg": (26.0 / 3.0) * n ** 3 / t_fused / 1e9,
        "effective_complex_rate_tflops": {"frobenius": 8.0 * n ** 3 / t_frob / 1e9, "zinv_lu": 8.0 * n ** 3 / t_zinv / 1e9,
                                          "note": "8 n^3 / t for both methods (SURVEY G12)"},
        "frob_over_zinv_time": t_frob / t_zinv, "fused_over_zinv_time": t_fused / t_zinv}
    if not big:
        t_rand = statistics.median(timed(lambda: fb.inv_rand(zr, mu=0.5, out=xr), reps, warm, True))
        extras["comparison_single_n"]["frobenius_randomized_ms"] = t_rand
    extras["threshold"] = {
        "n": n, "T_inv_ms": t_inv, "T_mult_ms": t_mult, "T_trmm_ms": t_trmm, "ratio_Tinv_Tmult": ratio,
        "lambda_measured": lam, "paper_threshold_1_plus_lambda_over_2": 1.0 + lam / 2.0,
        "paper_threshold_lambda_half": 1.25, "paper_threshold_lambda_one": 1.5, "r_z": r_z,
        "break_even_literal_lambda1": (3.0 / (r_z - 2)) if r_z > 2 else None,
        "break_even_fused_lambda": ((2 + lam) / (r_z - 2)) if r_z > 2 else None,
        "predicted_frob_faster": bool(r_z > 2 and ratio > 3.0 / (r_z - 2)),
        "measured_frob_faster": bool(t_frob < t_zinv),
        "predicted_fused_faster": bool(r_z > 2 and ratio > (2 + lam) / (r_z - 2)),
        "measured_fused_faster": bool(t_fused < t_zinv),
        "note": ("Thm 5.1 (P:L468-477): Frobenius beats complex LU iff T_inv/T_mult > 1 + lambda/2 when "
                 "T_zinv = 4 T_inv; with the measured r_z = T_zinv/T_inv the break-even is (2 + lambda)/(r_z - 2) "
                 "(lambda = 1 for the literal path, the measured lambda for NEXT-1)")}
    if isinstance(wl, Batched):
        cmp = {}
        z64 = torch.from_numpy(synth.batch(64, 16384, seed=0)).to(dev)
        for nn, zz in ((32, wl.parts[0][1]), (64, z64), (128, wl.parts[1][1])):
            tb_f = statistics.median(timed(lambda: fb.inv_batched(zz), 3, 1, False))
            tb_z = statistics.median(timed(lambda: fb.zinv_batched(zz), 3, 1, False))
            cnt = int(zz.shape[0])
            cmp[f"n{nn}"] = {"count": cnt, "frob_ms": tb_f, "zinv_lu_ms": tb_z, "frob_over_zinv_time": tb_f / tb_z,
                             "frob_inverses_per_s": cnt / tb_f * 1e3, "zinv_inverses_per_s": cnt / tb_z * 1e3,
                             "frob_tflops_alg": 10.0 * nn ** 3 * cnt / tb_f / 1e9,
                             "zinv_tflops_alg": 8.0 * nn ** 3 * cnt / tb_z / 1e9}
        extras["batched_comparison"] = cmp
    # NEXT-4: HPD inversion -- Alg 6 vs complex Cholesky Alg 8, and Thm 6.2's T_pinv / T_mult vs 7/6
    nh = min(n, 4096)
    zh = torch.from_numpy(synth.hpd(nh, seed=rank)).to(dev)
    xh = torch.empty_like(zh)
    t_h6 = statistics.median(timed(lambda: fb.hpd_inv(zh, out=xh, check=False), 3, 1, True))
    t_h8 = statistics.median(timed(lambda: fb.zhpd_inv(zh, out=xh, check=False), 3, 1, True))
    hpd = {"n": nh, "frob_hpd_alg6_ms": t_h6, "complex_cholesky_alg8_ms": t_h8, "alg6_over_alg8_time": t_h6 / t_h8}
    if hasattr(fb, "dpoinv"):
        ar = zh.real.contiguous()
        ai = torch.empty_like(ar)
        cm2 = torch.empty_like(ar)
        t_pinv = statistics.median(timed(lambda: fb.dpoinv(ar, out=ai), 3, 1, True))
        t_m2 = statistics.median(timed(lambda: fb.dgemm(ar, ai, cm2), 3, 1, True))
        hpd.update({"T_pinv_ms": t_pinv, "T_mult_ms": t_m2, "ratio_Tpinv_Tmult": t_pinv / t_m2,
                    "paper_threshold": 7.0 / 6.0, "predicted_alg6_faster": bool(t_pinv / t_m2 > 7.0 / 6.0),
                    "measured_alg6_faster": bool(t_h6 < t_h8),
                    "note": "Thm 6.2 (P:L847-871): Alg 6/7 beats complex Cholesky inversion iff T_pinv/T_mult > 7/6"})
    extras["hpd_comparison"] = hpd
    # GEMM engine (DMMA) at the n x n x n shape of the three Frobenius GEMMs
    ach = 2.0 * n ** 3 / t_mult / 1e9
    extras["roofline_gemm"] = {"bound": "tensor", "kernel": "gemm_kernel<double> (DMMA m8n8k4), n x n x n",
                               "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                               "peak_source": peak_src}
    # dominant kernel of the timed step: a separate instrumented pass (CUDA events recorded by the
    # library on the stream each kernel is launched on), never inside the timed region
    fbi.profile_enable(True)
    nprof = 2 if big else max(2, min(args.steps, 5))
    pw = timed(wl.step, nprof, 1, wl.flush)
    prof = fbi.profile_read()
    fbi.profile_enable(False)
    if prof:
        steps_prof = len(pw) + 1
        groups = _kernel_groups(prof)
        name, d = max(groups.items(), key=lambda kv: kv[1]["total_ms"])
        avg_ms = d["total_ms"] / max(1, d["launches"])
        ach_k = d["flops"] / max(1, d["launches"]) / (avg_ms * 1e-3) / 1e12
        tensor = name.startswith("gemm") or name.startswith("lu_update2") or name.startswith("lu_next2")
        pk, pk_src = (peak, peak_src) if tensor else fp64_alu_peak()
        traffic, tsrc = _traffic_for(name, getattr(wl, "n", None))
        extras["roofline"] = {
            "bound": "tensor" if tensor else "alu", "kernel": name, "achieved": ach_k, "peak": pk,
            "unit": "TFLOP/s", "frac": ach_k / pk, "traffic": traffic, "traffic_source": tsrc,
            "peak_source": pk_src,
            "flops_per_launch": d["flops"] / max(1, d["launches"]), "avg_launch_ms": avg_ms,
            "launches_per_step": d["launches"] / steps_prof,
            "share_of_step": d["total_ms"] / steps_prof / statistics.median(pw),
            "algorithmic": ("2 n^3 flop per launch (each of C = X^-1 Y, M = X + Y C, Im = -C Re is one n x n x n "
                            "GEMM launch)" if name.startswith("gemm_kernel<double> Frob") else
                            "the library's per-launch algorithmic flop count (DESIGN.md section 6)")}
        if name.startswith("lu_panel2"):
            # a pivot chain: report cycles per column against a latency floor built from the measured
            # primitive latencies (3 x REDUX chain 72, dependent LDS 38,
            # __syncthreads 36, DSMEM st.async + mbarrier round trip 519, DFMA 11, reciprocal 4 x DFMA)
            cluster = name.startswith("lu_panel2c")
            floor = 72 + (519 if cluster else 36) + 38 + 72 + 38 + 44 + 11
            cyc = avg_ms * 1e-3 * 1.965e9 / 32  # one launch = one 32-column step, cycles at the 1965 MHz clock
            extras["roofline"]["chain"] = {
                "cycles_per_column": cyc, "floor_cycles_per_column": floor, "frac": floor / cyc,
                "floor_basis": ("per column: warp argmax (3 dependent REDUX), " +
                                ("DSMEM candidate push + mbarrier round trip" if cluster else "__syncthreads") +
                                ", block argmax over the warp candidates (LDS + 3 REDUX), pivot-row read (LDS), "
                                "reciprocal (4 dependent DFMA), next column's update (DFMA); measured primitive "
                                "latencies, tools/lat_probe.cu / tools/dsmem_probe.cu")}
        extras["kernel_profile"] = {k: {"launches_per_step": v["launches"] / steps_prof,
                                        "ms_per_step": v["total_ms"] / steps_prof,
                                        "tflops": v["flops"] / (v["total_ms"] * 1e-3) / 1e12 if v["total_ms"] else None}
                                    for k, v in sorted(groups.items(), key=lambda kv: -kv[1]["total_ms"])}
        extras["role_profile"] = {k: {"launches_per_step": v["launches"] / steps_prof,
                                      "ms_per_step": v["total_ms"] / steps_prof}
                                  for k, v in prof.items() if k.startswith("step:")}
    # end to end through the host-buffer C-ABI call (H2D and D2H inside the timed region)
    ne2e = max(2, min(args.steps // 2, 3 if big else 10))
    e2e = timed(wl.e2e_step, ne2e, 1, False)
    e2e_ms = fdist.max_over_ranks(statistics.median(e2e), dev)
    extras["e2e"] = {"value": units_all / wl.units * 1e3 / e2e_ms if isinstance(wl, SingleMatrix) else units_all * 1e3 / e2e_ms,
                     "unit": UNIT, "h2d_bytes_per_step": int(wl.bytes_h2d()), "d2h_bytes_per_step": int(wl.bytes_d2h()),
                     "mode": wl.e2e_mode}
    if hasattr(wl, "e2e_pipelined"):
        kk = max(4, args.steps)
        got = wl.e2e_pipelined(kk)  # warm-up (and pinned buffers)
        if got:
            reps_ = []
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                wl.e2e_pipelined(kk)
                e1.record(stream)
                torch.cuda.synchronize()
                reps_.append(e0.elapsed_time(e1) / got)
            pm = fdist.max_over_ranks(statistics.median(reps_), dev)
            single = extras["e2e"]
            extras["e2e"] = {"value": units_all / wl.units * 1e3 / pm, "unit": UNIT,
                             "h2d_bytes_per_step": int(wl.bytes_h2d()), "d2h_bytes_per_step": int(wl.bytes_d2h()),
                             "mode": f"frob_inv_host_many over {got} distinct matrices per call: the host->device copy "
                                     f"of matrix i+1 and the device->host copy of matrix i-1 overlap inversion i",
                             "single_call": {"value": single["value"], "mode": single["mode"]}}
            if wl.flush:
                extras["e2e"]["l2"] = ("not flushed between the matrices of one pipelined call (distinct inputs; "
                                       "the device-resident value flushes L2 before every step)")
    return extras


if __name__ == "__main__":
    main()
