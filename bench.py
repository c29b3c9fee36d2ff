#!/usr/bin/env python
"""bench.py -- throughput of the whole hot path of arXiv 1509.04863 Algorithm 1
(fold -> template fold -> correlation -> argmax -> CRT) on B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5] [--impl reference]

One process per GPU (torchrun for N > 1).  Default workload cfg5: ONE signal of
N = 2^31 samples split into contiguous chunks over the ranks (strong scaling);
each rank folds its chunk, the partial folds are summed in place by one NCCL
all-reduce, the correlation is split by output blocks (SingleSignal,
paper_1509_04863_b200/single.py).  The batch workloads (cfg1-cfg4) shard
independent (signal, template) pairs with no data-path collective (weak
scaling, global pair indices rank*B + b); a step = one tm_run over the rank's
whole batch with inputs resident in HBM.
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
    # SURVEY 8(d) companions of the cfg4 K sweep (the K^2/log K transition)
    "cfg4c": dict(N=2 ** 24, K=32768, B=64, dtype="int8", noise=0.2, seed=4,
                  desc="cfg4 companion: N=2^24, K=32768, batch 64, +-1 int8, 20% flips"),
    "cfg4d": dict(N=2 ** 24, K=65536, B=64, dtype="int8", noise=0.2, seed=4,
                  desc="cfg4 companion: N=2^24, K=65536, batch 64, +-1 int8, 20% flips"),
    # PAPER.md Table 2's shape through the fp32 path (four-step FFT, L2 = 2^17)
    "t2": dict(N=2 ** 26, K=65536, B=8, dtype="float32", noise=0.5, seed=26,
               desc="Table 2 shape: N=2^26, K=2^16, batch 8, fp32 N(0,1), template noise sigma 0.5"),
    # one signal split into contiguous row-aligned chunks over the ranks (strong scaling)
    "cfg5": dict(N=2 ** 31, K=65536, B=1, dtype="int8", noise=0.05, seed=5, single=True,
                 desc="cfg5: one signal N=2^31 (+-1 int8, 2 GiB), K=65536, 5% flips, split over the GPUs; "
                      "partial folds summed by one NCCL all-reduce"),
}
EV_EVERY = 20  # timed steps between two stage-event samples (an event between two launches also ends their PDL overlap)
METRIC = "signal Gsamples/s matched (1/2/4/8 B200) and % of HBM roofline; match success rate"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def sample_steps(steps: int):
    """Timed steps that carry stage events: every EV_EVERY-th (at least two samples when
    steps >= 4), never step 0 (the first step after the warm-up's synchronize is not
    representative of the steady state)."""
    every = min(EV_EVERY, max(2, steps // 2))
    return [i for i in range(steps) if i % every == every - 1] or [steps - 1]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS),
                    help="cfg5 (default): the largest configuration, one 2 GiB signal, split over the ranks")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="oracle cpu_baseline budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--strategy", type=int, default=1, choices=[1, 2],
                    help="1: D_{M+K} (P:152, default); 2: Block Phi of Theorem 2 (P:159-177, TM_BLOCK)")
    ap.add_argument("--no-stage-events", action="store_true", help="A/B only: no per-step stage events")
    ap.add_argument("--no-cfg1", action="store_true", help="skip the cfg1 latency sample")
    ap.add_argument("--fused-reduce", action="store_true",
                    help="cfg5, world > 1: combine the partial folds in the fold epilogue (tm_fold_reduce into "
                         "symmetric memory / NVLS multicast, SURVEY 8(f) f4(iii)) instead of an NCCL all-reduce")
    ap.add_argument("--pipeline", type=int, default=0,
                    help="staged paths on one GPU: buffer sets of the two-stream step pipeline (tm.Pipeline / "
                         "SingleSignal(depth=)); 1 = every step strictly on one stream; 0 = the measured-best "
                         "default (3 for the single signal, 2 for batches)")
    ap.add_argument("--ref-seconds", type=float, default=150.0,
                    help="--impl reference: CPU budget of the timed steps (each step is whole pairs)")
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


NOMINAL_HBM_GBS = 8000.0  # BASELINE.json north_star "~8 TB/s"


def read_ceiling(tm, buf, stream, reps: int = 5):
    """Live read-only streaming ceiling on this box (tm_probe_read_bw: a cp.async.bulk
    ring over `buf`, one CTA per SM), best of `reps`, GB/s."""
    import torch
    nbytes = buf.numel() * buf.element_size()
    if nbytes < (256 << 20):   # too small to stream at bandwidth (cfg1): no live ceiling
        return None
    best = None
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tm.probe_read_bw(buf, stream=stream)
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None or ms < best else best
    return (nbytes // (32 * 1024) * 32 * 1024) / (best * 1e-3) / 1e9


def peak_denominators(ceiling):
    peak, _ = measured_peaks()
    d = {"nominal_8000": NOMINAL_HBM_GBS, "measured_copy": peak}
    if ceiling:
        d["read_ceiling_live"] = ceiling
    return d


def roofline_block(bound, achieved, kernel_ms, alg_bytes, kernel, traffic, ceiling):
    peak, src = measured_peaks()
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": kernel, "algorithmic_bytes_per_launch": alg_bytes,
            "peak_source": src, "kernel_ms": kernel_ms,
            "frac_by_denominator": {k: achieved / v for k, v in peak_denominators(ceiling).items()},
            "read_ceiling_gbs": ceiling}


def step_stats(per_step, mean_ms):
    xs = sorted(per_step)
    return {"mean": mean_ms, "median": statistics.median(xs), "min": xs[0], "max": xs[-1], "n": len(xs)}


def cfg1_latency(tm, dev, reps: int = 200):
    """cfg1 (N=4096, K=256, one pair): tm_run latency, each call bracketed by its own
    events (latency-bound); median / min / max in microseconds."""
    import torch
    wl = WORKLOADS["cfg1"]
    plan = tm.Plan(wl["N"], wl["K"], seed=wl["seed"])
    x, t, k0 = plan.generate(0, 1, wl["noise"], device=dev)
    ws = plan.workspace(1, dev)
    res = torch.empty((1, 2), dtype=torch.int32, device=dev)
    k = torch.empty(1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    for _ in range(10):
        plan.run(x, t, residues=res, k=k, ws=ws, stream=s)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record(s)
        plan.run(x, t, residues=res, k=k, ws=ws, stream=s)
        b.record(s)
    torch.cuda.synchronize()
    us = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return {"workload": wl["desc"], "unit": "us", "median": statistics.median(us), "min": us[0], "max": us[-1],
            "reps": reps, "path": tm.RUN_PATHS.get(plan.run_path(1)), "k_equals_k0": bool(int(k[0]) == int(k0[0]))}


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
    """The reference arm of this tier: the CPU oracle as it stands (single thread)
    on the same workload; each step is whole pairs (cfg5: the whole 2^31-sample
    pair), stopping early once --ref-seconds of timed CPU work is spent so the run
    ends within minutes.  Rank 0 only; other ranks exit without work."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np

    import oracle
    import tmgen
    oracle.build()
    cores, model = cpu_info()
    N, K = wl["N"], wl["K"]
    fn = oracle.ftm_block if args.strategy == 2 else oracle.ftm
    dt = np.int8 if wl["dtype"] == "int8" else np.float32
    warm = 0 if wl.get("single") else min(args.warmup, 3)   # a warm-up of a 40 s CPU pair buys nothing
    times = []
    pair = 0
    for i in range(warm + max(args.steps, 1)):
        x, t, _ = tmgen.batch(wl["seed"], 0 if wl.get("single") else pair, 1, N, K, wl["noise"], dtype=dt)
        t0 = time.perf_counter()
        fn(x[0], t[0], want_vectors=False)
        el = time.perf_counter() - t0
        del x
        pair += 1
        if i >= warm:
            times.append(el)
            if sum(times) >= args.ref_seconds:
                break
    spent = sum(times)
    rate = len(times) * N / spent / 1e9
    sample = (f"{len(times)} timed step(s) of {args.steps} requested, each one whole pair of {wl['desc']} "
              f"(host-generated by tmgen), {spent:.1f} s single-threaded; stopped at the {args.ref_seconds:.0f} s "
              f"budget" if len(times) < args.steps else
              f"{len(times)} step(s), each one whole pair of {wl['desc']} (host-generated), {spent:.1f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "Gsamples/s", "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": warm, "ms_per_step": spent / len(times) * 1e3,
        "higher_is_better": True, "scaling": "strong" if wl.get("single") else "weak", "vs_baseline": None,
        "dtype": "i8" if wl["dtype"] == "int8" else "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "N": N, "K": K, "batch": wl["B"],
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
    # inputs_stable: x and t are written before the timed region and never again, so
    # consecutive launches may stream x before their predecessor completes (PDL)
    plan = tm.Plan(N, K, seed=wl["seed"], dtype=wl["dtype"], block=args.strategy == 2, inputs_stable=True)
    stream = torch.cuda.current_stream()
    # inputs resident in HBM: this rank's pairs [rank*B, rank*B + B)
    x, t, k0 = plan.generate(rank * B, B, wl["noise"], device=dev)
    ws = plan.workspace(B, dev)
    residues = torch.empty((B, 2), dtype=torch.int32, device=dev)
    k = torch.empty(B, dtype=torch.int64, device=dev)
    torch.cuda.synchronize()

    path = plan.run_path(B)
    # staged paths: consecutive steps pipelined over two streams (the fold of step i+1
    # concurrent with the correlation of step i; tm.Pipeline).  The fused path
    # overlaps the two inside its one kernel.
    if args.pipeline == 0:
        args.pipeline = 2
    pipe = tm.Pipeline(plan, B, depth=args.pipeline, device=dev) if args.pipeline > 1 and path in (0, 1) else None

    def step():
        if pipe is not None:
            pipe.step(x, t, stream=stream)
        else:
            plan.run(x, t, residues=residues, k=k, ws=ws, stream=stream)

    def drain():
        if pipe is not None:
            pipe.drain(stream)

    for _ in range(max(args.warmup, 3)):
        step()
    drain()
    torch.cuda.synchronize()

    # ---- timed region: K steps.  Stage events (tm_profile_events) on every
    # EV_EVERY-th step only: each event record costs ~2.7 us of GPU time.
    # (pipelined: the sampled steps run tm_run on the caller's stream, which records the marks)
    nev = 2 if path == 2 else 5   # fused: before / after the one kernel
    ev_steps = sample_steps(args.steps) if not args.no_stage_events else []
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
                drain()   # the sampled step runs alone, in order on the caller's stream
                keep = tm.profile_events(ev[i])
                plan.run(x, t, residues=residues, k=k, ws=ws, stream=stream)
                tm.profile_events(None)
            else:
                step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        drain()
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

    # ---- per-step spread: a second pass with an event at every step boundary (the
    # events end the PDL overlap of consecutive steps, so this pass is slightly
    # slower than the headline pass above; it reports the spread, not the value)
    bnd = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    bnd[0].record(stream)
    for i in range(args.steps):
        step()
        bnd[i + 1].record(stream)
    drain()
    torch.cuda.synchronize()
    per_step = [bnd[i].elapsed_time(bnd[i + 1]) for i in range(args.steps)]
    if pipe is not None:   # the pipelined steps' results equal the one-stream tm_run's
        rp, kp = pipe._slots[pipe.last_slot]["residues"], pipe._slots[pipe.last_slot]["k"]
        if ev:
            assert torch.equal(kp, k) and torch.equal(rp, residues), "pipelined step differs from tm_run"
        residues, k = rp, kp
    ceiling = read_ceiling(tm, x, stream)

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
        "roofline": roofline_block("hbm", achieved, fold_ms, fold_bytes, kernel, traffic, ceiling),
        "run_path": tm.RUN_PATHS.get(path, str(path)),
        "pipeline": (f"depth {args.pipeline}: the fold of step i+1 (caller's stream) concurrent with the correlation "
                     f"of step i (side stream), tm.Pipeline" if pipe is not None else "none (one stream)"),
        "stage_ms": ({"fused_kernel": stage_mean[0]} if nev == 2 else
                     {"fold": stage_mean[0], "fold_template": stage_mean[1], "correlate_argmax": stage_mean[2],
                      "crt": stage_mean[3]}),
        "stage_events": f"on {len(ev)} of {args.steps} timed steps (steps {sorted(ev)[:3]}...)"
                        + ("; a sampled step runs tm_run alone on the caller's stream after a drain" if pipe else ""),
        "host_enqueue_ms_per_step": host_ms,
        "step_hbm_frac": (B * N * bx / (ms_max / args.steps * 1e-3) / 1e9) / peak,
        "step_hbm": {kk: B * N * bx / (ms_max / args.steps * 1e-3) / 1e9 / v
                     for kk, v in peak_denominators(ceiling).items()},
        "step_ms": step_stats(per_step, ms_max / args.steps),
        "success_rate": success,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
    }
    if world == 1 and not args.no_cfg1 and args.workload != "cfg1":
        line["cfg1_latency"] = cfg1_latency(tm, dev)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_single_signal(args, wl, rank, world, local, dev):
    """cfg5: one signal split over the ranks through the library's
    SingleSignal: each rank folds its chunk, the flat y1 || y2 buffer is summed in
    place by one all-reduce, the correlation is split by output blocks and the
    16-byte keys MAX-reduced (world > 1); every rank ends with the same k."""
    import torch
    import torch.distributed as dist

    import paper_1509_04863_b200 as tm
    from paper_1509_04863_b200 import dist as tmdist
    from paper_1509_04863_b200.single import SingleSignal

    N, K = wl["N"], wl["K"]
    plan = tm.Plan(N, K, seed=wl["seed"], dtype=wl["dtype"], block=args.strategy == 2, inputs_stable=True)
    stream = torch.cuda.current_stream()
    reducer = None
    if args.fused_reduce and world > 1:
        from paper_1509_04863_b200.single import SymmReducer
        reducer = SymmReducer()
    # one GPU: consecutive signals pipelined over two streams (SingleSignal(depth=)); with
    # ranks every step stays on one stream, the collectives between its stages
    depth = (args.pipeline or 3) if world == 1 and reducer is None else 1
    ss = SingleSignal(plan, rank, world, device=dev, reducer=reducer, depth=depth)
    off, ln = ss.offset, ss.length
    x, t, k0 = plan.generate(0, 1, wl["noise"], offset=off, length=ln, device=dev)
    torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        ss.step(x, t, stream=stream)
    ss.drain(stream)
    torch.cuda.synchronize()
    # stage events on every EV_EVERY-th timed step only (an event between two launches
    # ends their PDL overlap: with events at every step the cfg5 step read 0.376 ms
    # instead of 0.357); the per-step spread comes from a second pass below
    ev_steps = sample_steps(args.steps)
    ev = {i: [torch.cuda.Event(enable_timing=True) for _ in range(4)] for i in ev_steps}
    for e4 in ev.values():  # torch creates the CUDA event lazily on first record
        for e in e4:
            e.record(stream)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = tm.launch_count()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(args.steps):
            if i in ev:   # the sampled step runs alone (pipelined: no other step's kernels beside it)
                ss.drain(stream)
                ss.step(x, t, stream=stream, events=ev[i])
                ss.drain(stream)
            else:
                ss.step(x, t, stream=stream)
        ss.drain(stream)
        stop.record(stream)
        torch.cuda.synchronize()
    launches = tm.launch_count() - l0
    if world > 1:
        dist.barrier()
    ms_max = tmdist.max_over_ranks(start.elapsed_time(stop), device=dev)
    st = [statistics.mean(e[i].elapsed_time(e[i + 1]) for e in ev.values()) for i in range(3)]
    fold_ms = tmdist.max_over_ranks(st[0], device=dev)
    # per-step spread: a second pass with an event at every step boundary (slightly
    # slower than the headline pass: the events end the overlap of consecutive steps)
    bnd = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    torch.cuda.synchronize()
    bnd[0].record(stream)
    for i in range(args.steps):
        ss.step(x, t, stream=stream)
        bnd[i + 1].record(stream)
    ss.drain(stream)
    torch.cuda.synchronize()
    per_step = [bnd[i].elapsed_time(bnd[i + 1]) for i in range(args.steps)]
    res_dev, k_dev = ss.residues.clone(), ss.k.clone()
    ceiling = read_ceiling(tm, x, stream)
    # e2e: every step copies this rank's chunk from pinned host memory, runs the
    # same library step and reads k back
    e2e = None
    if args.e2e_steps > 0:
        xh = torch.empty((1, ln), dtype=x.dtype, pin_memory=True)
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
            _, kk = ss.step(xd, t, stream=stream)
            ss.drain(stream)   # (pipelined: k is written on the side stream)
            kh.copy_(kk, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = tmdist.max_over_ranks(e0.elapsed_time(e1), device=dev)
        assert int(kh[0]) == int(k_dev[0]), "e2e k differs from the device-resident run"
        e2e = {"value": N * args.e2e_steps / (e_ms * 1e-3) / 1e9, "unit": "Gsamples/s",
               "h2d_bytes_per_step": ln * x.element_size(), "d2h_bytes_per_step": 8, "steps": args.e2e_steps,
               "path": "pinned host chunk -> device copy -> SingleSignal.step -> k to pinned host, per step"}
        del xh, xd
    success = float((k_dev == k0).double().item())
    if rank == 0:
        bx = x.element_size()
        fold_bytes = ln * bx + (plan.len_y1 + plan.len_y2) * 4
        achieved = fold_bytes / (fold_ms * 1e-3) / 1e9
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cfg5_oracle_baseline(wl, plan, int(k_dev[0]), tuple(res_dev[0].tolist()))
        value = N * args.steps / (ms_max * 1e-3) / 1e9
        step_bytes = N * bx / world
        line = {
            "metric": METRIC, "value": value, "unit": "Gsamples/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "i8" if wl["dtype"] == "int8" else "f32",
            "data": "synthetic (seeded counter-based generator, chunks generated on each rank's device)",
            "config": {"workload": wl["desc"], "N": N, "K": K, "M1": plan.M1, "M2": plan.M2, "chunk_samples": ln,
                       "parallelism": f"sequence split over {world} rank(s)"
                                      + ((f" + fold epilogue adding y1||y2 ({ss.reduce_bytes} B) into every rank's "
                                          f"symmetric buffer ({'NVLS multicast' if reducer.destinations()[2] else 'peer'})"
                                          if reducer is not None else
                                          f" + in-place all-reduce of y1||y2 ({ss.reduce_bytes} B)")
                                         + " + correlation split by output blocks + all-reduce MAX of 16 B keys"
                                         if world > 1 else ""),
                       "pipeline": (f"depth {depth}: the fold of step i+1 (caller's stream) concurrent with the "
                                    f"correlation of step i (side stream)" if depth > 1 else "none (one stream)"),
                       "l2": "no flush: per-rank input > 126 MB L2"},
            "roofline": roofline_block("hbm", achieved, fold_ms, fold_bytes,
                                       "tm_fold (zero_i32 + fold_pm1_tma + fold_finalize)",
                                       traffic_of(args.workload) if world == 1 else None, ceiling),
            "stage_ms": {"fold": st[0], "allreduce": st[1], "correlate_match": st[2]},
            "stage_events": f"on {len(ev)} of {args.steps} timed steps (steps {sorted(ev)[:3]}...)"
                            + ("; a sampled step runs alone, drained before and after" if depth > 1 else ""),
            "step_ms": step_stats(per_step, ms_max / args.steps),
            "step_hbm": {k: step_bytes / (ms_max / args.steps * 1e-3) / 1e9 / v
                         for k, v in peak_denominators(ceiling).items()},
            "success_rate": success, "k": int(k_dev[0]), "k0": int(k0.item()),
            "residues": res_dev[0].tolist(),
            "cpu_baseline": cpu, "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": launches,
        }
        if world == 1 and not args.no_cfg1:
            line["cfg1_latency"] = cfg1_latency(tm, dev)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cfg5_oracle_baseline(wl, plan, k_gpu, res_gpu):
    """The oracle as it stands (single thread) on the whole cfg5 pair: host-generated
    x (2 GiB) and t, Eq. 2 folds of both moduli, direct correlations, argmax, CRT.
    Its k and residues are also checked against the GPU's (the full-size parity of
    SURVEY 8(c.3))."""
    import numpy as np

    import oracle
    import tmgen
    N, K = wl["N"], wl["K"]
    xs = tmgen.signal(wl["seed"], 0, N)
    ts = tmgen.template(wl["seed"], 0, N, K, wl["noise"])
    t0 = time.perf_counter()
    o = oracle.ftm(xs, ts, want_vectors=False)
    dt = time.perf_counter() - t0
    cores, model = cpu_info()
    del xs
    return {"value": N / dt / 1e9, "unit": "Gsamples/s", "cores": 1, "kind": "oracle",
            "sample": f"the whole cfg5 pair (N=2^31, K=65536): Eq. 2 folds of both moduli + direct correlations + "
                      f"argmax + CRT, {dt:.1f} s single-threaded",
            "seconds": dt, "host_cpus": cores, "cpu_model": model,
            "oracle_k": int(o["k"]), "oracle_residues": list(o["residues"]),
            "matches_gpu": bool(o["k"] == k_gpu and tuple(o["residues"]) == tuple(res_gpu))}


if __name__ == "__main__":
    main()
