#!/usr/bin/env python
"""Benchmark of the rdFFT hot path on B200 (driver contract: one JSON line).

Step — one pass of every §8(a) row over one batch:
  bca_fwd   RoBERTa-base adapter  (configs[2]: T = 32 x 512, d = 768, p = 256, bf16)
  bca_fwd   LLaMA2-7B adapter     (configs[3]: T = 8 x 2048, d = 4096, p = 1024, bf16)
  rdfft_fwd X = 2^20 vectors of n = 1024, bf16 (configs[1]; 2 GiB, in place)
  rdfft_packed_mul  X <- X (.) H  (H = rdFFT(delta_37): one all-pass filter spectrum, broadcast)
  rdfft_inv X in place
  bca_bwd   RoBERTa-base, then LLaMA2-7B (dx into its own buffer, dw fp32)
            [+ NCCL all_reduce(dw) when N > 1]
The 2 GiB transform traffic sits between every layer's forward and backward, and the LLaMA
backward (400 MB) between the RoBERTa backward and the next step's RoBERTa forward, so no BCA
operand is L2-resident when its kernel starts (inputs larger than L2 between reuses).
The filter has |H_k| = 1 and dx never overwrites g, so the data stay the same distribution over
any number of steps (the transforms are norm-preserving up to rounding).

N > 1 (launched with torchrun, or by `--gpus N` itself): configs[4] — a GLOBAL batch of 2^24
vectors of n = 1024 and 2^22 LLaMA-shape tokens, generated as 64 fixed seeded chunks (identical
global data for every N) and sharded contiguously over the ranks (strong scaling); the only
collective is the fp32 dw all-reduce.  `--workload cfg4` runs the same at N = 1.

value = the metric BASELINE.json names: in-place rdFFT fwd+inv GB/s (bf16, n = 1024) = algorithmic
bytes of rdfft_fwd + rdfft_inv over all ranks (2 * 2 n s per vector) / (max over ranks of their summed
device time); the BCA fwd+bwd ms per shape is reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "in-place rdFFT fwd+inv GB/s vs HBM peak (bf16, n=1024); BCA layer fwd+bwd ms"
N_FFT = 1024
BATCH = 1 << 20                      # configs[1]
CFG4_VECTORS = 1 << 24               # configs[4] global batch
CFG4_TOKENS = 1 << 22                # configs[4] BCA variant (SURVEY §8(d) cfg 5), global tokens
LLAMA = dict(name="llama2_7b", T=8 * 2048, d_in=4096, d_out=4096, p=1024)       # configs[3]
ROBERTA = dict(name="roberta_base", T=32 * 512, d_in=768, d_out=768, p=256)    # configs[2]
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s), only if MEASURED_PEAKS.json is absent


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ------------------------------------------------------------- CPU oracle
def cpu_oracle_rate(budget_s: float = 12.0, n: int = N_FFT):
    """Time the float64 oracle (as it stands) on rdfft_fwd + rdfft_inv of seeded
    n = 1024 vectors, chunk by chunk, for about `budget_s` seconds.  Returns GB/s
    in the metric's unit (algorithmic bf16 bytes of the same work) and the sample."""
    import oracle as o
    from paper_2511_01385_b200 import synth

    chunk = 1024
    done, t_used, i = 0, 0.0, 0
    while t_used < budget_s and i < 1024:
        x = synth.randn((chunk, n), seed=7000 + i, dtype="bf16").double().numpy()
        t0 = time.perf_counter()
        p = o.rdfft_fwd(x)
        o.rdfft_inv(p)
        t_used += time.perf_counter() - t0
        done += chunk
        i += 1
    gbs = done * 2 * (2 * n * 2) / t_used / 1e9
    return gbs, t_used, done, cpu_threads()


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max([d.get("num_threads", 1) for d in info if d.get("user_api") == "blas"] or [os.cpu_count()])
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def worked_example(dev=None):
    """configs[0]: the n = 8 fp32 batch-4 worked example (SURVEY §8(d) cfg 1: rows delta_0, ones,
    cos(2 pi t / 8), 1..8) — fwd + inv round trip; the CPU oracle timed in ms, the GPU in us per
    launch pair (launch-bound), both checked against the closed-form packed spectra (P1)."""
    import math

    import numpy as np

    import oracle as o

    n = 8
    t = np.arange(n)
    x = np.stack([(t == 0).astype(float), np.ones(n), np.cos(2 * np.pi * t / n), t + 1.0])
    r2 = math.sqrt(2.0)
    want = np.array([[1, 1, 1, 1, 1, 0, 0, 0], [8, 0, 0, 0, 0, 0, 0, 0], [0, 4, 0, 0, 0, 0, 0, 0],
                     [36, -4, -4, -4, -4, 4 * (r2 - 1), 4, 4 * (r2 + 1)]], dtype=float)
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        pk = o.rdfft_fwd(x)
        back = o.rdfft_inv(pk)
    cpu_ms = (time.perf_counter() - t0) * 1e3 / reps
    out = {"config": "configs[0]: n=8 fp32, batch 4 (rows delta_0, ones, cos(2 pi t/8), 1..8)",
           "oracle_ms_fwd_inv": cpu_ms, "oracle_max_abs_err_vs_closed_form": float(np.abs(pk - want).max()),
           "oracle_round_trip_max_abs_err": float(np.abs(back - x).max()), "cpu_threads": cpu_threads()}
    if dev is not None:
        import torch

        from paper_2511_01385_b200 import rdfft as R

        xd = torch.tensor(x, dtype=torch.float32, device=dev)
        R.rdfft_fwd(xd)
        torch.cuda.synchronize()
        got = xd.double().cpu().numpy()
        R.rdfft_inv(xd)
        torch.cuda.synchronize()
        rt = xd.double().cpu().numpy()
        st = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(20):
            R.rdfft_fwd(xd)
            R.rdfft_inv(xd)
        greps = 1000
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(greps):
            R.rdfft_fwd(xd)
            R.rdfft_inv(xd)
        e1.record(st)
        torch.cuda.synchronize()
        out.update({"gpu_us_fwd_inv": 1e3 * e0.elapsed_time(e1) / greps,
                    "gpu_max_abs_err_vs_closed_form": float(np.abs(got - want).max()),
                    "gpu_round_trip_max_abs_err": float(np.abs(rt - x).max()),
                    "gpu_note": "launch-bound: two kernel launches per round trip (CUDA events over 1000 reps)"})
    return out


# --------------------------------------------------------------- reference arm
def arm_config(args, world: int) -> dict:
    """The workload both arms report (the reference arm times the oracle on a sample of it)."""
    if cfg4_mode(args, world):
        return {"workload": f"configs[4]: rdFFT fwd+packed_mul+inv on a global batch of 2^{CFG4_VECTORS.bit_length() - 1}"
                            f" x n={N_FFT} bf16 + BCA fwd+bwd LLaMA2-7B adapter (d=4096, p=1024) on 2^"
                            f"{CFG4_TOKENS.bit_length() - 1} global tokens, both sharded over {world} GPU(s)",
                "n": N_FFT, "global_batch": CFG4_VECTORS, "global_tokens": CFG4_TOKENS, "bca": [LLAMA],
                "parallelism": f"dp{world}", "data_chunks": 64,
                "l2": "inputs larger than L2 (every tensor >= 2 GiB per GPU)"}
    return {"workload": f"configs[1]+[2]+[3]: rdFFT fwd+packed_mul+inv on 2^{args.batch.bit_length() - 1} x "
                        f"n={N_FFT} bf16 per GPU + BCA fwd+bwd RoBERTa-base (T=16384, d=768, p=256) and "
                        f"LLaMA2-7B (T=16384, d=4096, p=1024) adapters, bf16",
            "n": N_FFT, "batch_per_gpu": args.batch, "bca": [ROBERTA, LLAMA], "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 between reuses (2 GiB transform buffer between every BCA forward and "
                  "its backward; the 400 MB LLaMA backward between the RoBERTa backward and forward)"}


def cfg4_mode(args, world):
    return world > 1 or args.workload == "cfg4"


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_oracle_rate(budget_s=min(2.0, budget))
    secs, vecs, threads = 0.0, 0, 1
    for _ in range(args.steps):
        _gbs, t, done, threads = cpu_oracle_rate(budget_s=budget)
        secs += t
        vecs += done
    value = vecs * 2 * (2 * N_FFT * 2) / secs / 1e9
    sample = (f"oracle rdfft_fwd+rdfft_inv (float64 O(n^2) DFT + pack / IDFT, numpy BLAS) on {vecs} seeded "
              f"bf16-rounded vectors of n={N_FFT} out of the workload, {args.steps} steps of ~{budget:.0f} s")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(1, args.steps),
            "higher_is_better": True, "scaling": "strong" if cfg4_mode(args, world) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": arm_config(args, world),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- GPU arm
def rfft_flops(n):
    """Exact flop count of the paper's radix-2 real FFT: per stage m, each of the
    n/2m blocks costs 2 (k = 0) + 10 per general four-slot group (complex multiply 6 + 4 adds);
    the m = 1 stage is n/2 butterflies of 2 adds.  19 976 at n = 1024."""
    total, m = n, 2
    while m < n:
        total += (n // (2 * m)) * (2 + 10 * (m // 2 - 1))
        m *= 2
    return total


def bca_work(sh, T):
    """Algorithmic bytes and flops of one BCA forward / backward launch over T tokens."""
    s = 2
    p, q_in, q_out = sh["p"], sh["d_in"] // sh["p"], sh["d_out"] // sh["p"]
    prod = q_out * q_in * (8 * (p // 2 - 1) + 4)
    F = rfft_flops(p)
    return {"fwd": (T * (sh["d_in"] + sh["d_out"]) * s, T * ((q_in + q_out) * F + prod)),
            "bwd": (T * (2 * sh["d_in"] + sh["d_out"]) * s, T * ((2 * q_in + q_out) * F + 2 * prod))}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2511_01385_b200 import build, synth
    from paper_2511_01385_b200 import dist as Dd
    from paper_2511_01385_b200 import rdfft as R

    world, rank, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)  # before the process group: NCCL binds each rank to its own GPU
    dev = torch.device("cuda", local)
    if world > 1:
        # NCCL over NVLink on the box; RDFFT_DIST_BACKEND=gloo lets the N > 1 logic run with several
        # ranks on one GPU (a functional check of sharding / barriers / max-over-ranks / dw all-reduce)
        backend = os.environ.get("RDFFT_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group(backend, device_id=dev)
        else:
            dist.init_process_group(backend)
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    R._lib()

    n, s = N_FFT, 2
    cfg4 = cfg4_mode(args, world)
    if cfg4:
        total = args.global_batch or CFG4_VECTORS
        ttot = args.global_tokens or CFG4_TOKENS
        lo, hi = Dd.shard_range(total, rank, world)
        tlo, thi = Dd.shard_range(ttot, rank, world)
        X = synth.randn_rows(total, (n,), lo, hi, seed=1000, dtype="bf16", device=dev)
        shapes = [dict(LLAMA, T=thi - tlo)]
        bca_data = []
        sh = LLAMA
        q_in, q_out = sh["d_in"] // sh["p"], sh["d_out"] // sh["p"]
        xa = synth.randn_rows(ttot, (sh["d_in"],), tlo, thi, seed=2000, dtype="bf16", device=dev)
        w = synth.randn((q_out, q_in, sh["p"]), seed=2999, dtype="bf16", device=dev, std=sh["d_in"] ** -0.5)
        g = synth.randn_rows(ttot, (sh["d_out"],), tlo, thi, seed=3000, dtype="bf16", device=dev)
        ya = torch.empty((thi - tlo, sh["d_out"]), dtype=torch.bfloat16, device=dev)
        bca_data.append((sh["name"], xa, w, g, ya, ya, torch.empty((q_out, q_in, sh["p"]), dtype=torch.float32,
                                                                   device=dev)))  # dx reuses y's buffer
        nvec_total = total
    else:
        X = synth.randn((args.batch, n), seed=1000 + rank, dtype="bf16", device=dev)
        shapes = [ROBERTA, LLAMA]
        bca_data = []
        for i, sh in enumerate(shapes):
            q_in, q_out = sh["d_in"] // sh["p"], sh["d_out"] // sh["p"]
            xa, w, g = synth.bca_inputs(sh["T"], sh["d_in"], sh["d_out"], sh["p"], seed=2000 + 10 * i + rank,
                                        dtype="bf16", device=dev)
            bca_data.append((sh["name"], xa, w, g, torch.empty((sh["T"], sh["d_out"]), dtype=torch.bfloat16, device=dev),
                             torch.empty((sh["T"], sh["d_in"]), dtype=torch.bfloat16, device=dev),
                             torch.empty((q_out, q_in, sh["p"]), dtype=torch.float32, device=dev)))
        nvec_total = world * args.batch
    nvec = X.shape[0]
    # filter spectrum H = rdFFT(delta_37): |H_k| = 1 in every bin (an all-pass filter, a circular shift),
    # so the step's repeated fwd -> (.) H -> inv keeps X's distribution
    Hf = torch.zeros((1, n), dtype=torch.bfloat16, device=dev)
    Hf[0, 37] = 1
    R.rdfft_fwd(Hf)
    stream = torch.cuda.current_stream(dev)

    names = ([f"bca_fwd_{b[0]}" for b in bca_data] + ["rdfft_fwd", "packed_mul", "rdfft_inv"] +
             [f"bca_bwd_{b[0]}" for b in bca_data] + (["allreduce_dw"] if world > 1 else []))

    def step(ev=None):
        k = 0

        def mark():
            nonlocal k
            if ev is not None:
                ev[k].record(stream)
            k += 1
        mark()
        for _nm, xa, w, g, ya, dxa, dw in bca_data:
            R.bca_fwd(xa, w, ya)
            mark()
        R.rdfft_fwd(X)
        mark()
        R.rdfft_packed_mul(X, Hf)
        mark()
        R.rdfft_inv(X)
        mark()
        for _nm, xa, w, g, ya, dxa, dw in bca_data:
            R.bca_bwd(xa, w, g, dxa, dw)
            mark()
        if world > 1:
            for b in bca_data:
                Dd.allreduce_dw(b[6])  # the one real exchange: sum of per-shard weight gradients
            mark()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    nev = len(names) + 1
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    launches0 = R.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        # ~1 ms of device-side spin BEFORE t_start: the host enqueues the first steps while the GPU
        # spins, so no timed segment waits on a host launch (without it the first step's first
        # segments absorb the ~13-30 us host cost of each ctypes call: RoBERTa bca_fwd read 0.047 ms
        # in the bench against 0.035 ms for the same kernel after a 2 GiB transform, tools/diag_seg.py)
        torch.cuda._sleep(2_000_000)
        t_start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = R.launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    seg = {nm: sum(e[i].elapsed_time(e[i + 1]) for e in evs) / args.steps for i, nm in enumerate(names)}
    i_fwd, i_inv = names.index("rdfft_fwd"), names.index("rdfft_inv")

    def allmax(v):
        return Dd.max_over_ranks(v, device=dev)

    fwdinv_ms = allmax(sum(e[i_fwd].elapsed_time(e[i_fwd + 1]) + e[i_inv].elapsed_time(e[i_inv + 1])
                           for e in evs) / args.steps)
    total_ms = allmax(total_ms)
    seg = {k: allmax(v) for k, v in seg.items()}
    bytes_fft_all = 2 * n * s * nvec_total      # one direction, all ranks (algorithmic: read n + write n)
    value = 2 * bytes_fft_all / (fwdinv_ms * 1e-3) / 1e9
    hbm, peak_src = peaks()

    # ---- end to end through the C-ABI with HOST buffers (copies inside the timed region): pinned host
    # rows -> rdfft_filter_host (H2D, rdfft_fwd, packed_mul, rdfft_inv, D2H on two streams) -> host
    e2e = None
    if not args.no_e2e:
        e_rows = min(nvec, args.e2e_rows)
        Xh = torch.empty((e_rows, n), dtype=torch.bfloat16, pin_memory=True)
        Xh.copy_(X[:e_rows])
        work = torch.empty((2 * args.e2e_chunk, n), dtype=torch.bfloat16, device=dev)
        strs = [torch.cuda.Stream(dev) for _ in range(2)]
        R.rdfft_filter_host(Xh, work, Hf, streams=strs)  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_steps = max(1, min(args.steps, 5))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            R.rdfft_filter_host(Xh, work, Hf, streams=strs)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = allmax(e0.elapsed_time(e1) / e2e_steps)
        e2e = {"value": world * 2 * (2 * n * s * e_rows) / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": e_rows * n * s, "d2h_bytes_per_step": e_rows * n * s, "ms_per_step": e2e_ms,
               "path": f"C-ABI rdfft_filter_host: pinned host [{e_rows} x {n}] bf16 -> H2D -> rdfft_fwd -> "
                       f"rdfft_packed_mul -> rdfft_inv -> D2H, {args.e2e_chunk}-row chunks on 2 streams "
                       f"(per GPU; same GB/s unit as value: fwd+inv algorithmic bytes)"}
        del Xh, work

    # ---- rooflines: transforms / packed_mul against HBM; BCA against the FP32 FMA issue peak
    clocks = sampler.summary()
    fp32_peak = 148 * 128 * 2 * (clocks.get("sm_max_mhz") or 1965) * 1e6 / 1e12
    kern = {"rdfft_fwd": (2 * n * s * nvec, None), "rdfft_inv": (2 * n * s * nvec, None),
            "packed_mul": (2 * n * s * nvec, None)}
    for (nm, xa, *_rest), sh in zip(bca_data, shapes):
        wk = bca_work(sh, xa.shape[0])
        kern[f"bca_fwd_{nm}"] = wk["fwd"]
        kern[f"bca_bwd_{nm}"] = wk["bwd"]
    rooflines = {}
    for k, (b, f) in kern.items():
        ach = b / (seg[k] * 1e-3) / 1e9
        r = {"ms": seg[k], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
             "bytes": b, "achieved_GBps": ach}
        if f is not None:
            a = f / (seg[k] * 1e-3) / 1e12
            r.update({"bound": "alu", "achieved": a, "peak": fp32_peak, "unit": "TFLOP/s", "frac": a / fp32_peak,
                      "flops": f, "hbm_frac": ach / hbm})
        rooflines[k] = r
    dom = max(kern, key=lambda k: seg[k])
    roofline = {"kernel": dom, "bound": rooflines[dom]["bound"], "achieved": rooflines[dom]["achieved"],
                "peak": rooflines[dom]["peak"], "unit": rooflines[dom]["unit"], "frac": rooflines[dom]["frac"],
                "traffic": ncu_traffic(dom, nvec), "peak_source": peak_src, "bytes_per_launch": kern[dom][0],
                "ms_per_launch": seg[dom]}

    cpu = wex = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, t, done, threads = cpu_oracle_rate(budget_s=args.cpu_budget)
        cpu = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle",
               "sample": f"float64 oracle (numpy BLAS) rdfft_fwd+rdfft_inv on {done} seeded vectors of n={n} "
                         f"({t:.1f} s), same algorithmic-bytes unit", **host_info()}
        wex = worked_example(dev)

    if rank == 0:
        bca_ms = {b[0]: {"fwd_ms": seg[f"bca_fwd_{b[0]}"], "bwd_ms": seg[f"bca_bwd_{b[0]}"],
                         "fwd_bwd_ms": seg[f"bca_fwd_{b[0]}"] + seg[f"bca_bwd_{b[0]}"], "tokens_per_gpu": b[1].shape[0]}
                  for b in bca_data}
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if cfg4 else "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": arm_config(args, world),
            "frac_of_hbm_peak": value / (world * hbm), "hbm_peak_GBps": hbm,
            "transforms_per_s": 2 * nvec_total / (fwdinv_ms * 1e-3),
            "bca": bca_ms, "bca_fwd_bwd_ms": bca_ms[LLAMA["name"]]["fwd_bwd_ms"],
            "segments_ms": seg, "rooflines": rooflines, "roofline": roofline,
            "cpu_baseline": cpu, "worked_example": wex, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ncu_traffic(kernel, batch):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed `ncu --set full`
    capture (profiles/ncu_traffic.json, written by tools/ncu_summary.py).  The transform and
    packed-multiply captures run at a smaller batch; their traffic is scaled to this launch."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(kernel)
        if not e:
            return None
        t = float(e["dram_bytes_per_launch"])
        if kernel in ("rdfft_fwd", "rdfft_inv", "packed_mul"):
            t *= batch / float(e.get("batch", 1 << 18))
        return t
    except Exception:  # noqa: BLE001
        return None


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto", choices=["auto", "cfg4"],
                    help="auto: configs[1]+[2]+[3] at N = 1, configs[4] at N > 1; cfg4: configs[4] at any N")
    ap.add_argument("--batch", type=int, default=BATCH, help="vectors per GPU (configs[1] mode)")
    ap.add_argument("--global-batch", type=int, default=0, help="configs[4] global vectors (default 2^24)")
    ap.add_argument("--global-tokens", type=int, default=0, help="configs[4] global BCA tokens (default 2^22)")
    ap.add_argument("--e2e-rows", type=int, default=1 << 20)
    ap.add_argument("--e2e-chunk", type=int, default=1 << 16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: launch the ranks ourselves (same as the driver's torchrun command)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
