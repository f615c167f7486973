#!/usr/bin/env python
"""Benchmark of the rdFFT hot path on B200 (driver contract: one JSON line).

Step — one pass of every §8(a) row over one batch:
  bca_fwd   LLaMA2-7B BCA adapter: T = 8 x 2048 tokens, d = 4096, p = 1024, bf16
  rdfft_fwd X = 2^20 vectors of n = 1024, bf16 (2 GiB, in place)
  rdfft_packed_mul  X <- X (.) H   (H one packed filter spectrum, broadcast)
  rdfft_inv X in place
  bca_bwd   same layer (dx overwrites g in place, dw fp32) [+ NCCL all_reduce(dw) when N > 1]
The 2 GiB transform traffic between bca_fwd and bca_bwd flushes the 126 MB L2.

value = the metric BASELINE.json names: in-place rdFFT fwd+inv GB/s (bf16,
n = 1024) = algorithmic bytes of rdfft_fwd + rdfft_inv (2 * 2 n s per vector,
all ranks) / (max over ranks of their summed device time); the BCA fwd+bwd ms
is reported beside it.  Weak scaling: every rank runs the full per-GPU batch.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "in-place rdFFT fwd+inv GB/s vs HBM peak (bf16, n=1024); BCA layer fwd+bwd ms"
N_FFT = 1024
BATCH = 1 << 20
BCA = dict(T=8 * 2048, d_in=4096, d_out=4096, p=1024)
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
            time.sleep(0.02)

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
    import numpy as np

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
    threads = cpu_threads()
    return gbs, t_used, done, threads, np.__version__


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max([d.get("num_threads", 1) for d in info if d.get("user_api") == "blas"] or [os.cpu_count()])
    except Exception:  # noqa: BLE001
        return os.cpu_count()


# --------------------------------------------------------------- reference arm
def arm_config(batch: int, world: int) -> dict:
    """The workload both arms report (the reference arm times the oracle on a sample of it)."""
    T, d_in, p = BCA["T"], BCA["d_in"], BCA["p"]
    return {"workload": f"rdFFT fwd+packed_mul+inv on 2^{batch.bit_length() - 1} x n={N_FFT} bf16 per GPU "
                        f"+ BCA fwd+bwd LLaMA2-7B adapter (T={T}, d={d_in}, p={p}, bf16)",
            "n": N_FFT, "batch_per_gpu": batch, "bca": BCA, "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (2 GiB transform buffer per GPU between BCA fwd and bwd)"}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2511_01385_b200 import synth  # noqa: F401  (input generator only)

    budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_oracle_rate(budget_s=min(2.0, budget))
    rates, secs, vecs = [], 0.0, 0
    for _ in range(args.steps):
        gbs, t, done, threads, _v = cpu_oracle_rate(budget_s=budget)
        rates.append(gbs)
        secs += t
        vecs += done
    value = vecs * 2 * (2 * N_FFT * 2) / secs / 1e9
    sample = (f"oracle rdfft_fwd+rdfft_inv (float64 O(n^2) DFT + pack / IDFT) on {vecs} seeded bf16-rounded "
              f"vectors of n={N_FFT} out of the 2^20-vector workload, {args.steps} steps of ~{budget:.0f} s")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": arm_config(args.batch, world),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# -------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2511_01385_b200 import build, synth
    from paper_2511_01385_b200 import dist as Dd
    from paper_2511_01385_b200 import rdfft as R

    world, rank, local = dist_env()
    if world > 1:
        # NCCL over NVLink on the box; RDFFT_DIST_BACKEND=gloo lets the N > 1 logic run with several
        # ranks on one GPU (a functional check of barriers / max-over-ranks / the dw all-reduce)
        dist.init_process_group(os.environ.get("RDFFT_DIST_BACKEND", "nccl"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    R._lib()

    n, batch, s = N_FFT, args.batch, 2
    T, d_in, d_out, p = BCA["T"], BCA["d_in"], BCA["d_out"], BCA["p"]
    q_in, q_out = d_in // p, d_out // p
    # Seeded inputs; rank r draws its own shard (weak scaling), generated on device.
    X = synth.randn((batch, n), seed=1000 + rank, dtype="bf16", device=dev)
    Hf = synth.randn((1, n), seed=999, dtype="bf16", device=dev)
    xa, w, g = synth.bca_inputs(T, d_in, d_out, p, seed=2000 + rank, dtype="bf16", device=dev)
    ya = torch.empty((T, d_out), dtype=torch.bfloat16, device=dev)
    dw = torch.empty((q_out, q_in, p), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    names = ["bca_fwd", "rdfft_fwd", "packed_mul", "rdfft_inv", "bca_bwd"] + (["allreduce_dw"] if world > 1 else [])

    def step(ev=None):
        def mark(i):
            if ev is not None:
                ev[i].record(stream)
        mark(0)
        R.bca_fwd(xa, w, ya)
        mark(1)
        R.rdfft_fwd(X)
        mark(2)
        R.rdfft_packed_mul(X, Hf)
        mark(3)
        R.rdfft_inv(X)
        mark(4)
        R.bca_bwd(xa, w, g, g, dw)  # dx overwrites grad_output in place
        mark(5)
        if world > 1:
            Dd.allreduce_dw(dw)  # the one real exchange: sum of per-shard weight gradients
            mark(6)

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

    def allmax(v):
        return Dd.max_over_ranks(v, device=dev)

    total_ms = allmax(total_ms)
    seg = {k: allmax(v) for k, v in seg.items()}
    fwdinv_ms = allmax(sum(e[1].elapsed_time(e[2]) + e[3].elapsed_time(e[4]) for e in evs) / args.steps)
    bytes_fft = 2 * n * s * batch  # one direction, algorithmic (read n + write n reals per vector)
    value = world * 2 * bytes_fft / (fwdinv_ms * 1e-3) / 1e9
    hbm, peak_src = peaks()

    # ---- end to end through the public API with host buffers (copies timed): pinned host batch
    # streamed through the device in row chunks on two streams (H2D / transforms / D2H overlap)
    e2e = None
    if not args.no_e2e:
        from paper_2511_01385_b200 import pipeline as PL

        Xh = torch.empty((batch, n), dtype=torch.bfloat16, pin_memory=True)
        Xh.copy_(X)
        strs = [torch.cuda.Stream(dev) for _ in range(2)]
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = max(1, min(args.steps, 5))
        PL.fwd_inv_host(Xh, X, streams=strs)  # warm-up
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(e2e_steps):
            PL.fwd_inv_host(Xh, X, streams=strs)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = allmax(e0.elapsed_time(e1) / e2e_steps)
        e2e = {"value": world * 2 * bytes_fft / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": batch * n * s, "d2h_bytes_per_step": batch * n * s,
               "ms_per_step": e2e_ms,
               "path": "pinned host -> device -> rdfft_fwd -> rdfft_inv -> pinned host, 2^16-row chunks on 2 streams "
                       "(paper_2511_01385_b200.pipeline.fwd_inv_host)"}
        del Xh

    # ---- roofline for the dominant kernel (largest share of the step)
    kern_bytes = {"rdfft_fwd": bytes_fft, "rdfft_inv": bytes_fft, "packed_mul": 2 * n * s * batch,
                  "bca_fwd": T * (d_in + d_out) * s, "bca_bwd": T * (2 * d_in + d_out) * s}
    # BCA is bound by FP32 issue, not HBM: algorithmic flops (the paper's radix-2 count
    # F(p) per transform, 8 flops per complex multiply-add) against the FP32 FMA peak
    # 148 SMs x 128 lanes x 2 flops x the SM clock (B200_PROFILING.md unit counts)
    q_in, q_out = d_in // p, d_out // p
    prod = q_out * q_in * (8 * (p // 2 - 1) + 4)
    kern_flops = {"bca_fwd": T * ((q_in + q_out) * rfft_flops(p) + prod),
                  "bca_bwd": T * ((2 * q_in + q_out) * rfft_flops(p) + 2 * prod)}
    rooflines = {}
    for k, b in kern_bytes.items():
        ach = b / (seg[k] * 1e-3) / 1e9
        rooflines[k] = {"ms": seg[k], "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                        "bytes": b, "achieved_GBps": ach}
    clocks = sampler.summary()
    fp32_peak = 148 * 128 * 2 * (clocks.get("sm_max_mhz") or 1965) * 1e6 / 1e12
    for k, f in kern_flops.items():
        ach = f / (seg[k] * 1e-3) / 1e12
        rooflines[k].update({"bound": "alu", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s",
                             "frac": ach / fp32_peak, "flops": f,
                             "hbm_frac": rooflines[k]["achieved_GBps"] / hbm})
    dom = max(kern_bytes, key=lambda k: seg[k])
    traffic = ncu_traffic(dom, batch)
    roofline = {"kernel": dom, "bound": rooflines[dom]["bound"], "achieved": rooflines[dom]["achieved"],
                "peak": rooflines[dom]["peak"], "unit": rooflines[dom]["unit"], "frac": rooflines[dom]["frac"],
                "traffic": traffic, "peak_source": peak_src, "bytes_per_launch": kern_bytes[dom],
                "ms_per_launch": seg[dom]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, t, done, threads, _ = cpu_oracle_rate(budget_s=args.cpu_budget)
        cpu = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle",
               "sample": f"float64 oracle rdfft_fwd+rdfft_inv on {done} seeded vectors of n={n} "
                         f"({t:.1f} s), same algorithmic-bytes unit"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": arm_config(batch, world),
            "frac_of_hbm_peak": value / (world * hbm), "hbm_peak_GBps": hbm,
            "transforms_per_s": world * 2 * batch / (fwdinv_ms * 1e-3),
            "bca_fwd_ms": seg["bca_fwd"], "bca_bwd_ms": seg["bca_bwd"],
            "bca_fwd_bwd_ms": seg["bca_fwd"] + seg["bca_bwd"],
            "segments_ms": seg, "rooflines": rooflines, "roofline": roofline,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def rfft_flops(n):
    """Exact flop count of the paper's radix-2 real FFT: per stage m, each of the
    n/2m blocks costs 2 (k = 0) + 10 per general four-slot group (complex multiply 6 + 4 adds);
    the m = 1 stage is n/2 butterflies of 2 adds.  19 976 at n = 1024."""
    total, m = n, 2
    while m < n:
        total += (n // (2 * m)) * (2 + 10 * (m // 2 - 1))
        m *= 2
    return total


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=BATCH)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
