#!/usr/bin/env python
"""Benchmark of the B200 batched PA-aware precoder solver.

Headline (BASELINE.json): precoders/s of the 20-layer unfolded PGD at K = 8
users, M = 64 antennas — SURVEY §8d config 2: 65,536 realizations per GPU,
CN(0,1) channels with per-user gains log-uniform over 20 dB, seeded projected
layer parameters, W0 = 0. One step = one pass of the fused kernel over the
GPU's batch plus the reduction of the summary statistics (an NCCL all-reduce
when N > 1). Weak scaling: every rank owns its own 65,536 realizations
(global indices rank*B .. rank*B + B - 1).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
  python bench.py --impl reference ...   # the reference CPU path (FP64 oracle)

Rank 0 prints one JSON line. `value` is device-timed (CUDA events, barrier and
synchronize on both sides, max over ranks) with H resident in HBM; `e2e` is the
same metric through the C ABI host-buffer entry point
(ufpgd_gpu_unfolded_forward_host) from pinned host memory, H2D and D2H inside
the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "precoders/sec (20-layer unfolded PGD, M=64,K=8) at 1/2/4/8 B200; % of roofline"
UNIT = "precoders/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-other-configs", action="store_true")
    return ap.parse_args()


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------
# clocks during the timed region (NVML)
# --------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.period = period_s
        self.samples, self.reasons = [], 0
        self.ok = False
        try:
            import pynvml as N
            import torch

            N.nvmlInit()
            self.N = N
            p = torch.cuda.get_device_properties(device_index)
            try:
                bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
                self.h = N.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # NVML missing: report it, keep benchmarking
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.N.nvmlDeviceGetClockInfo(self.h, self.N.NVML_CLOCK_SM))
                self.reasons |= self.N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()

    def report(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "nvml")}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# --------------------------------------------------------------------------
# the reference CPU path (FP64 oracle restatement; the reference cannot be
# built here — SURVEY §8c) — used by --impl reference and the cpu_baseline leg
# --------------------------------------------------------------------------
def reference_rate(w, H, lam, eta, steps, warmup, threads):
    from oracle import oracle as O

    for _ in range(warmup):
        O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode, threads=threads, want_W=False)
    t0 = time.perf_counter()
    for _ in range(steps):
        O.forward_batch_f32(H, w.c, lam, eta, w0_mode=w.w0_mode, threads=threads, want_W=False)
    return steps * len(H) / (time.perf_counter() - t0)


def clamped_layers(w):
    """Layers whose raw step mu_l was clamped by project_params (SURVEY §8d asks for the count)."""
    import paper_2304_12745_b200 as U

    raw_lam, raw_eta = U.layer_params(w.seed_p, w.L, w.K, w.M)
    _, eta = U.project_params(raw_lam, raw_eta, w.K, w.M)
    return int(np.count_nonzero(eta != raw_eta))


def cpu_baseline(w, H, lam, eta, seconds):
    from oracle import oracle as O

    threads = O.default_thread_count()
    n = min(len(H), 8192)
    sample = np.ascontiguousarray(H[:n])
    O.forward_batch_f32(sample[:512], w.c, lam, eta, w0_mode=w.w0_mode, threads=threads, want_W=False)
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        O.forward_batch_f32(sample, w.c, lam, eta, w0_mode=w.w0_mode, threads=threads, want_W=False)
        done += n
    rate = done / (time.perf_counter() - t0)
    # the same port on one core (SURVEY §8d asks for both), over a ~2 s sample
    one = sample[:256]
    done1, t1 = 0, time.perf_counter()
    while time.perf_counter() - t1 < min(2.0, seconds):
        O.forward_batch_f32(one, w.c, lam, eta, w0_mode=w.w0_mode, threads=1, want_W=False)
        done1 += len(one)
    rate1 = done1 / (time.perf_counter() - t1)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "single_core_value": rate1,
            "sample": f"{done} realizations ({n} distinct of the rank-0 cfg{w.config} batch, repeated for "
                      f">= {seconds:g} s): FP64 C++ restatement of unfolded.cpp:83-146 forward, "
                      f"restated parallel_for (parallel.cpp:25-59) over {threads} threads"}


def run_reference(args, world, rank):
    if rank != 0:
        return
    import paper_2304_12745_b200 as U
    from oracle import oracle as O

    w = U.CONFIGS[args.config]
    threads = O.default_thread_count()
    n = 8192 if w.kind == "unfolded" else 16
    H = U.make_inputs(w, 0, n)
    lam, eta = w.layer_params()
    rate = reference_rate(w, H, lam, eta, args.steps, args.warmup, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": n / rate * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name(), "sample_per_step": n},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{n} of the cfg{w.config} realizations per step; FP64 oracle restatement of the "
                                   "reference forward (Eigen-based reference not buildable here, SURVEY §8c)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our path
# --------------------------------------------------------------------------
def load_traffic(w):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        e = d.get(f"cfg{w.config}")
        return e["dram_bytes_per_launch"] if e else None
    except Exception:
        return None


def measured_peaks():
    """The driver-written MEASURED_PEAKS.json (HBM copy GB/s, cuBLAS bf16
    TFLOP/s on this pool's B200s), with B200_PROFILING.md's fallbacks."""
    peaks = {"hbm_gbs": 6547.8, "bf16_tflops": 1724.1, "source": "fallback"}
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        peaks.update({k: float(d[k]) for k in ("hbm_gbs", "bf16_tflops") if k in d})
        peaks["source"] = "MEASURED_PEAKS.json"
    except Exception:
        pass
    return peaks


def measure_other_configs(U, torch, local):
    """Device-timed throughput of the other BASELINE configs (parity-test cases,
    not bench lines): one warm-up launch, then CUDA-event timing, on the full
    seeded batches generated on the device (the reference draw,
    ufpgd_gpu_generate_channels)."""
    res = {}
    for cid in (1, 3, 4, 5):
        w = U.CONFIGS[cid]
        H = U.generate_channels_device(w.seed_h, w.seed_g, w.gain_db, 0, w.B, w.K, w.M, device=local)
        reps = 3 if cid in (3, 4, 5) else 200

        if w.kind == "pgd":
            def run():
                return U.pgd_fixed(H, w.lambda_pgd, w.L, w.c, power_steps=w.power_steps, w0_mode=w.w0_mode)
        else:
            lam, eta = w.layer_params()
            Wd = torch.empty_like(H)

            def run():
                return U.unfolded_forward(H, lam, eta, w.c, w0_mode=w.w0_mode, out=Wd)
        run()
        torch.cuda.synchronize()
        # Replay a CUDA graph of the call so config 1's ~25 us launch is not
        # timed as Python + ctypes host overhead; fall back to direct calls.
        graph = None
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                out = run()
            graph.replay()
            torch.cuda.synchronize()
        except Exception:
            graph = None
            torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            if graph is not None:
                graph.replay()
            else:
                out = run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        st = out["stats"].cpu().numpy()
        res[f"cfg{cid}"] = {"workload": w.name(), "ms_per_batch": ms, "precoders_per_s": w.B / ms * 1e3,
                            "tflops": w.flops_per_realization() * w.B / ms / 1e9, "diverged": int(st[2]),
                            "mean_active": float(st[1]) / w.B, "note": "full batch, device-generated",
                            "cuda_graph": graph is not None}
        tf = w.tensor_flops_per_realization()
        if tf is not None and os.environ.get("UFPGD_NO_MMA", "0") != "1":
            pk = measured_peaks()
            ach = tf * w.B / ms / 1e9
            res[f"cfg{cid}"]["kernel"] = "mma_kernel (tcgen05.mma kind::f16, TMEM accumulators, 3-term f16 split)"
            res[f"cfg{cid}"]["tensor"] = {"achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                                          "frac": ach / pk["bf16_tflops"],
                                          "peak_source": pk["source"] + " bf16_tflops (f16 runs at the bf16 rate)",
                                          "flops_per_realization": tf}
        del graph
        del H
        torch.cuda.empty_cache()
    return res


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2304_12745_b200 as U

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    w = U.CONFIGS[args.config]
    if w.kind != "unfolded":
        raise SystemExit("bench.py times the unfolded configs; see tools/quick_time.py for PGD")
    from paper_2304_12745_b200 import sharding

    first, B = sharding.weak_shard(rank, w.B)
    H_host = torch.from_numpy(U.make_inputs(w, first, B)).pin_memory()
    lam, eta = w.layer_params()
    Hd = H_host.to(dev, non_blocking=False)
    Wd = torch.empty_like(Hd)
    stream = torch.cuda.current_stream(dev)

    def step():
        out = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode, out=Wd)
        sharding.reduce_stats(out["stats"])  # the one collective: 3 doubles (N > 1)
        return out

    for _ in range(max(3, args.warmup)):
        out = step()
    torch.cuda.synchronize()
    peak_tflops, peak_ghz = U.fp32_peak(local)
    nominal_tflops = torch.cuda.get_device_properties(local).multi_processor_count * 128 * 2 * 1.965e9 / 1e12

    # ---- device-timed region ------------------------------------------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t_start.record(stream)
    for k in range(args.steps):
        ev[k][0].record(stream)
        out = U.unfolded_forward(Hd, lam, eta, w.c, w0_mode=w.w0_mode, out=Wd)
        ev[k][1].record(stream)
        sharding.reduce_stats(out["stats"])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.stop()
    ms_local = t_start.elapsed_time(t_end)
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    stats = out["stats"].cpu().numpy()
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    else:
        ms_total = ms_local
    value = world * B * args.steps / (ms_total * 1e-3)

    # ---- end to end through the C ABI host-buffer entry point ----------------
    W_host = torch.empty_like(H_host).pin_memory()
    Hn, Wn = H_host.numpy(), W_host.numpy()
    for _ in range(2):
        U.unfolded_forward_host(Hn, lam, eta, w.c, w0_mode=w.w0_mode, out=Wn, device=local)
    e2e_steps = max(3, args.steps // 5)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r = U.unfolded_forward_host(Hn, lam, eta, w.c, w0_mode=w.w0_mode, out=Wn, device=local)
        if world > 1:
            sharding.reduce_stats(torch.from_numpy(r["stats"]).to(dev))
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = world * B * e2e_steps / e2e_s
    elem = w.K * w.M * 8

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, H_host.numpy(), lam, eta, args.cpu_seconds)
    others = None
    if rank == 0 and world == 1 and not args.no_other_configs:
        others = measure_other_configs(U, torch, local)

    if rank == 0:
        peaks = measured_peaks()
        flops = w.flops_per_realization() * B
        achieved = flops / (kern_ms * 1e-3) / 1e12
        hbm_bytes = w.bytes_per_realization() * B
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded CN(0,1) channels via the reference generate_channel rule, "
                    f"{w.gain_db:g} dB log-uniform user gains, complex64; seeded projected layer params)",
            "config": {"workload": w.name(), "per_gpu_batch": B, "global_batch": world * B, "K": w.K,
                       "M": w.M, "layers": w.L, "w0": "zero", "parallelism": f"dp{world} (independent shards, "
                       "NCCL all-reduce of 3 statistics per step)" if world > 1 else "single GPU",
                       "l2": f"inputs larger than L2: H = {w.B * elem / 2**20:.0f} MiB per GPU > 126 MB L2; no flush",
                       "seeds": {"h": w.seed_h, "g": w.seed_g, "p": w.seed_p},
                       "layers_eta_clamped_by_projection": clamped_layers(w)},
            "roofline": {
                "bound": "fp32", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                "frac": achieved / peak_tflops, "traffic": load_traffic(w),
                "peak_source": "measured live: FFMA2 outer-product probe (the kernel's instruction form), "
                               f"SM clock {peak_ghz:.3f} GHz during the probe; MEASURED_PEAKS.json has no FP32 entry",
                "nominal_peak": nominal_tflops, "frac_of_nominal": achieved / nominal_tflops,
                "kernel": "fused_kernel<Team<8,64,4,4>> (+stats_finalize)", "kernel_ms": kern_ms,
                "flops_per_launch": flops,
                "flops_model": "(2L-2)*8*K^2*M + 10*K*M*L per realization (W0 = 0: neither layer-0 "
                               "contraction is computed — W0 H^T is zero and X' = -diag(c)); SURVEY §8d "
                               "counts 2L contractions",
                "hbm": {"achieved_GBps": hbm_bytes / (kern_ms * 1e-3) / 1e9, "peak_GBps": peaks["hbm_gbs"],
                        "frac": hbm_bytes / (kern_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                        "bytes_per_launch": hbm_bytes, "peak_source": peaks["source"] + " hbm_gbs"},
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": B * elem,
                    "d2h_bytes_per_step": B * elem + B * 4 + 24, "steps": e2e_steps,
                    "path": "ufpgd_gpu_unfolded_forward_host (pinned host H in, W + diverged + stats out)"},
            "gpu_launches": 2 * args.steps,
            "clocks": clocks.report(),
            "stats": sharding.summarize(stats, world * B),
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
