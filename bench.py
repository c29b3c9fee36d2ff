#!/usr/bin/env python
"""bench.py -- throughput of the whole hot path of arXiv 1509.04863 Algorithm 1
(fold -> template fold -> correlation -> argmax -> CRT) on B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--impl reference]

One process per GPU (torchrun for N > 1).  Independent (signal, template) pairs
shard across ranks with no data-path collective (weak scaling: every rank
folds its own batch of the configuration, global pair indices rank*B + b).
A step = one tm_run over the rank's whole batch with inputs resident in HBM.
Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle
(oracle/, the test-infrastructure checker) on a bounded sample instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: (N, K, batch, dtype, noise, seed)
WORKLOADS = {
    "cfg1": dict(N=4096, K=256, B=1, dtype="int8", noise=0.0, seed=1,
                 desc="cfg1: N=4096, K=256, batch 1, +-1 int8, noiseless"),
    "cfg2": dict(N=2 ** 20, K=4096, B=1024, dtype="int8", noise=0.1, seed=2,
                 desc="cfg2: N=2^20, K=4096, batch 1024, +-1 int8, 10% template bit flips"),
    "cfg3": dict(N=2 ** 22, K=8192, B=256, dtype="float32", noise=0.5, seed=3,
                 desc="cfg3: N=2^22, K=8192, batch 256, fp32 N(0,1), template noise sigma 0.5"),
    "cfg4a": dict(N=2 ** 24, K=4096, B=64, dtype="int8", noise=0.2, seed=4,
                  desc="cfg4: N=2^24, K=4096, batch 64, +-1 int8, 20% flips"),
    "cfg4b": dict(N=2 ** 24, K=8192, B=64, dtype="int8", noise=0.2, seed=4,
                  desc="cfg4: N=2^24, K=8192, batch 64, +-1 int8, 20% flips"),
    "cfg4": dict(N=2 ** 24, K=16384, B=64, dtype="int8", noise=0.2, seed=4,
                 desc="cfg4: N=2^24, K=16384, batch 64, +-1 int8, 20% flips"),
    # one signal split into contiguous row-aligned chunks over the ranks (strong scaling)
    "cfg5": dict(N=2 ** 31, K=65536, B=1, dtype="int8", noise=0.05, seed=5, single=True,
                 desc="cfg5: one signal N=2^31 (+-1 int8, 2 GiB), K=65536, 5% flips, split over the GPUs; "
                      "partial folds summed by one NCCL all-reduce"),
}
EV_EVERY = 20  # timed steps between two stage-event samples (an event between two launches also ends their PDL overlap)
METRIC = "signal Gsamples/s matched (1/2/4/8 B200) and % of HBM roofline; match success rate"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle cpu_baseline budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strategy", type=int, default=1, choices=[1, 2],
                    help="1: D_{M+K} (P:152, default); 2: Block Phi of Theorem 2 (P:159-177, TM_BLOCK)")
    ap.add_argument("--no-stage-events", action="store_true", help="A/B only: no per-step stage events")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def traffic_of(key):
    """dram read + write bytes per launch of the roofline kernel(s) from one ncu --set
    full capture (profiles/ncu_traffic.json), or None"""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tp):
        return None
    with open(tp) as f:
        return json.load(f).get(key)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, device_index: int, period: float = 0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._period = period
        self._idx = device_index
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self._idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                getattr(pynvml, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(pynvml, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(pynvml, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
            }

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, name in names.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    time.sleep(self._period)

            self._t = threading.Thread(target=loop, daemon=True)
            self._t.start()
        except Exception as e:  # NVML unavailable: report it
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


def oracle_rate(wl, budget_s: float, max_pairs: int | None = None, strategy: int = 1):
    """Time the CPU oracle (single thread, as it stands) on pairs of the same
    workload until the budget is spent.  Returns (Gsamples/s, pairs, seconds)."""
    import numpy as np

    import oracle
    import tmgen
    dt = np.int8 if wl["dtype"] == "int8" else np.float32
    N, K = wl["N"], wl["K"]
    done, spent = 0, 0.0
    while spent < budget_s and (max_pairs is None or done < max_pairs):
        x, t, _ = tmgen.batch(wl["seed"], done, 1, N, K, wl["noise"], dtype=dt)
        t0 = time.perf_counter()
        (oracle.ftm_block if strategy == 2 else oracle.ftm)(x[0], t[0], want_vectors=False)
        spent += time.perf_counter() - t0
        done += 1
    return done * N / spent / 1e9, done, spent


def run_reference(args, wl):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    cores, model = cpu_info()
    # each step: one pair of the workload through the oracle (a bounded sample)
    if args.warmup:
        oracle_rate(wl, float("inf"), max_pairs=min(args.warmup, 3), strategy=args.strategy)
    rate, pairs, spent = oracle_rate(wl, float("inf"), max_pairs=max(args.steps, 1), strategy=args.strategy)
    sample = f"{pairs} pair(s) of {wl['desc']} (one pair per step), host-generated by tmgen"
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "Gsamples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": spent / max(pairs, 1) * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "i8" if wl["dtype"] == "int8" else "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "N": wl["N"], "K": wl["K"], "batch": wl["B"],
                   "parallelism": "single CPU thread (oracle)", "strategy": args.strategy},
        "cpu_baseline": {"value": rate, "unit": "Gsamples/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cpus": cores, "cpu_model": model},
        "e2e": {"value": rate, "unit": "Gsamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    import paper_1509_04863_b200 as tm

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if wl.get("single"):
        return run_single_signal(args, wl, rank, world, local, dev)
    N, K, B = wl["N"], wl["K"], wl["B"]
    plan = tm.Plan(N, K, seed=wl["seed"], dtype=wl["dtype"], block=args.strategy == 2)
    stream = torch.cuda.current_stream()
    # inputs resident in HBM: this rank's pairs [rank*B, rank*B + B)
    x, t, k0 = plan.generate(rank * B, B, wl["noise"], device=dev)
    ws = plan.workspace(B, dev)
    residues = torch.empty((B, 2), dtype=torch.int32, device=dev)
    k = torch.empty(B, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    def step():
        plan.run(x, t, residues=residues, k=k, ws=ws, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps.  Stage events (tm_profile_events) on every
    # EV_EVERY-th step only: each event record costs ~2.7 us of GPU time.
    path = plan.run_path(B)
    nev = 2 if path == 2 else 5   # fused: before / after the one kernel
    ev_steps = [i for i in range(args.steps) if i % EV_EVERY == 0] if not args.no_stage_events else []
    ev = {i: [torch.cuda.Event(enable_timing=True) for _ in range(nev)] for i in ev_steps}
    for e5 in ev.values():  # torch creates the CUDA event lazily on first record
        for e in e5:
            e.record(stream)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = tm.launch_count()
    keep = None
    with ClockSampler(local) as clocks:
        start.record(stream)
        h0 = time.perf_counter()
        for i in range(args.steps):
            if i in ev:
                keep = tm.profile_events(ev[i])
                step()
                tm.profile_events(None)
            else:
                step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        stop.record(stream)
        torch.cuda.synchronize()
    launches = tm.launch_count() - launches0
    del keep
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    stage_ms = [[e[i].elapsed_time(e[i + 1]) for i in range(nev - 1)] for e in ev.values()] or [[0.0] * (nev - 1)]
    fold_ms = statistics.mean(s[0] for s in stage_ms)
    stage_mean = [statistics.mean(s[i] for s in stage_ms) for i in range(nev - 1)]
    t_ms = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_max = float(t_ms.item())
    succ = (k == k0).double().mean()
    if world > 1:
        dist.all_reduce(succ)
        succ /= world
    success = float(succ.item())

    # ---- end to end through tm_run_host: pinned host inputs, H2D + compute + D2H per step
    e2e = None
    if args.e2e_steps > 0:
        chunk = max(1, min(B, 64))
        xh = torch.empty((B, N), dtype=x.dtype, pin_memory=True)
        th = torch.empty((B, K), dtype=t.dtype, pin_memory=True)
        xh.copy_(x.cpu())
        th.copy_(t.cpu())
        kh = torch.empty(B, dtype=torch.int64, pin_memory=True)
        rh = torch.empty((B, 2), dtype=torch.int32, pin_memory=True)
        dx, dtt, dout, wsc = plan.run_host_buffers(B, chunk, dev)
        plan.run_host(xh, th, chunk, rh, kh, dx, dtt, dout, wsc, stream=stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            plan.run_host(xh, th, chunk, rh, kh, dx, dtt, dout, wsc, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
        assert torch.equal(kh.to(dev), k), "tm_run_host result differs from tm_run"
        bx = x.element_size()
        e2e = {"value": world * B * N * args.e2e_steps / (float(e_ms.item()) * 1e-3) / 1e9, "unit": "Gsamples/s",
               "h2d_bytes_per_step": B * (N + K) * bx, "d2h_bytes_per_step": B * (8 + 8),
               "steps": args.e2e_steps, "chunk_pairs": chunk}
        del xh, th, dx, dtt, dout, wsc

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    bx = x.element_size()
    peak, peak_src = measured_peaks()
    if path == 2:
        # fused kernel = the whole step: algorithmic bytes = x and t read once, k and
        # residues written once (y never needs to leave the chip)
        kernel = "fold_pm1_tma<4,0,1,TC> (fused fold + tensor-core correlation + argmax + CRT)"
        fold_bytes = B * (N + K) * bx + B * (8 + 8)
        tkey = args.workload + ":fused_tc"
    else:
        # fold kernel algorithmic bytes per launch: read x once + write y1, y2 once
        kernel = ("fold_f32_strips + fold_f32_finalize (tm_fold, fp32)" if wl["dtype"] == "float32"
                  else "fold_pm1_tma<4,0,1> (fold)")
        fold_bytes = B * N * bx + B * (plan.len_y1 + plan.len_y2) * 4
        tkey = args.workload
    achieved = fold_bytes / (fold_ms * 1e-3) / 1e9
    traffic = traffic_of(tkey)
    cpu = None
    if not args.no_cpu_baseline:
        cores, model = cpu_info()
        rate, pairs, spent = oracle_rate(wl, args.cpu_seconds, strategy=args.strategy)
        cpu = {"value": rate, "unit": "Gsamples/s", "cores": 1, "kind": "oracle",
               "sample": f"{pairs} pair(s) of {wl['desc']}, {spent:.1f} s single-threaded",
               "host_cpus": cores, "cpu_model": model}
    value = world * B * N * args.steps / (ms_max * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "Gsamples/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "i8" if wl["dtype"] == "int8" else "f32",
        "data": "synthetic (seeded counter-based generator, inputs generated on device)",
        "config": {"workload": wl["desc"], "N": N, "K": K, "batch_per_gpu": B, "M1": plan.M1, "M2": plan.M2,
                   "parallelism": f"dp{world} (independent pairs)",
                   "strategy": "2 (Block Phi, Theorem 2)" if args.strategy == 2 else "1 (D_{M+K}, P:152)",
                   "l2": f"no flush: per-step input {B * N * bx / 2**30:.2f} GiB > 126 MB L2"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": kernel,
                     "algorithmic_bytes_per_launch": fold_bytes, "peak_source": peak_src,
                     "kernel_ms": fold_ms},
        "run_path": tm.RUN_PATHS.get(path, str(path)),
        "stage_ms": ({"fused_kernel": stage_mean[0]} if nev == 2 else
                     {"fold": stage_mean[0], "fold_template": stage_mean[1], "correlate_argmax": stage_mean[2],
                      "crt": stage_mean[3]}),
        "stage_events": f"on {len(ev)} of {args.steps} timed steps (every {EV_EVERY}th)",
        "host_enqueue_ms_per_step": host_ms,
        "step_hbm_frac": (B * N * bx / (ms_max / args.steps * 1e-3) / 1e9) / peak,
        "success_rate": success,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_single_signal(args, wl, rank, world, local, dev):
    """cfg5: each rank folds its chunk of the one signal (global positions), the
    partial folds are summed with one all-reduce, every rank correlates/matches."""
    import torch
    import torch.distributed as dist

    import paper_1509_04863_b200 as tm
    from paper_1509_04863_b200 import dist as tmdist

    N, K = wl["N"], wl["K"]
    plan = tm.Plan(N, K, seed=wl["seed"], dtype=wl["dtype"], block=args.strategy == 2)
    stream = torch.cuda.current_stream()
    off, ln = tmdist.signal_chunks(N, plan.M1, world)[rank]
    x, t, k0 = plan.generate(0, 1, wl["noise"], offset=off, length=ln, device=dev)
    ws = plan.workspace(1, dev)
    y1 = torch.empty((1, plan.len_y1), dtype=torch.int32, device=dev)
    y2 = torch.empty((1, plan.len_y2), dtype=torch.int32, device=dev)
    res = torch.empty((1, 2), dtype=torch.int32, device=dev)
    k = torch.empty(1, dtype=torch.int64, device=dev)
    keys = torch.empty((1, 2), dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    def step(ev=None):
        if ev: ev[0].record(stream)
        plan.fold(x, offset=off, length=ln, y1=y1, y2=y2, accumulate=False, ws=ws, stream=stream)
        if ev: ev[1].record(stream)
        if world > 1:
            tmdist.allreduce_folds(y1, y2)
        if ev: ev[2].record(stream)
        if world > 1:  # split the correlation by outputs, MAX-reduce the keys
            plan.correlate_match_part(y1, y2, t, rank, world, keys=keys, ws=ws, stream=stream)
            tmdist.allreduce_max_keys(keys)
            plan.match_keys(keys, residues=res, k=k, stream=stream)
        else:
            plan.correlate_match(y1, y2, t, residues=res, k=k, ws=ws, stream=stream)
        if ev: ev[3].record(stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = tm.launch_count()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            step(ev[i])
        stop.record(stream)
        torch.cuda.synchronize()
    launches = tm.launch_count() - l0
    if world > 1:
        dist.barrier()
    ms_max = tmdist.max_over_ranks(start.elapsed_time(stop), device=dev)
    st = [statistics.mean(e[i].elapsed_time(e[i + 1]) for e in ev) for i in range(3)]
    fold_ms = tmdist.max_over_ranks(st[0], device=dev)
    # e2e: the chunk copied from pinned host memory every step, k read back
    e2e = None
    if args.e2e_steps > 0:
        xh = torch.empty((1, ln), dtype=torch.int8, pin_memory=True)
        xh.copy_(x.cpu())
        xd = torch.empty_like(x)
        kh = torch.empty(1, dtype=torch.int64, pin_memory=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            xd.copy_(xh, non_blocking=True)
            plan.fold(xd, offset=off, length=ln, y1=y1, y2=y2, ws=ws, stream=stream)
            if world > 1:
                tmdist.allreduce_folds(y1, y2)
                plan.correlate_match_part(y1, y2, t, rank, world, keys=keys, ws=ws, stream=stream)
                tmdist.allreduce_max_keys(keys)
                plan.match_keys(keys, residues=res, k=k, stream=stream)
            else:
                plan.correlate_match(y1, y2, t, residues=res, k=k, ws=ws, stream=stream)
            kh.copy_(k, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = tmdist.max_over_ranks(e0.elapsed_time(e1), device=dev)
        e2e = {"value": N * args.e2e_steps / (e_ms * 1e-3) / 1e9, "unit": "Gsamples/s",
               "h2d_bytes_per_step": ln, "d2h_bytes_per_step": 8, "steps": args.e2e_steps}
        del xh, xd
    success = float((k == k0).double().item())
    if rank == 0:
        peak, peak_src = measured_peaks()
        fold_bytes = ln + (plan.len_y1 + plan.len_y2) * 4
        achieved = fold_bytes / (fold_ms * 1e-3) / 1e9
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            # the oracle's Eq. 2 fold of cfg5 alone is minutes of CPU: report the
            # oracle on a bounded sample (the fold of 2^-6 of the signal's rows)
            import numpy as np
            import time as _t
            import oracle
            import tmgen
            n_s = N // 64
            xs = tmgen.signal(wl["seed"], 0, N, lo=0, length=n_s)
            t0 = _t.perf_counter()
            oracle.fold(xs, plan.M1, K)
            oracle.fold(xs, plan.M2, K)
            dt = _t.perf_counter() - t0
            cpu = {"value": n_s / dt / 1e9, "unit": "Gsamples/s", "cores": 1, "kind": "oracle",
                   "sample": f"oracle Eq. 2 folds (M1 and M2) of the first 2^25 samples of the cfg5 signal "
                             f"taken as a signal of length 2^25 (correlation excluded: K=65536 is minutes of "
                             f"CPU), {dt:.1f} s"}
        line = {
            "metric": METRIC, "value": N * args.steps / (ms_max * 1e-3) / 1e9, "unit": "Gsamples/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i8",
            "data": "synthetic (seeded counter-based generator, chunks generated on each rank's device)",
            "config": {"workload": wl["desc"], "N": N, "K": K, "M1": plan.M1, "M2": plan.M2, "chunk_samples": ln,
                       "parallelism": f"sequence split over {world} rank(s) + NCCL all-reduce of y1||y2 "
                                      f"({(plan.len_y1 + plan.len_y2) * 4} B)"
                                      + (f"; correlation split by output blocks + all-reduce MAX of 16 B keys"
                                         if world > 1 else ""),
                       "l2": "no flush: per-rank input > 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic_of(args.workload) if world == 1 else None,
                         "kernel": "tm_fold (fold_pm1_tma + fold_finalize)",
                         "algorithmic_bytes_per_launch": fold_bytes, "peak_source": peak_src, "fold_ms": fold_ms},
            "stage_ms": {"fold": st[0], "allreduce": st[1], "correlate_match": st[2]},
            "success_rate": success, "k": int(k.item()), "k0": int(k0.item()),
            "cpu_baseline": cpu, "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
