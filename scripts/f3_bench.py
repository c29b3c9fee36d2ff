"""SURVEY 8(f) f3 (the section-3.5 acquisition shape): one folded signal against
many templates.  Times tm_correlate_many (steps 4-9 for every template, the
folded signal read at stride 0) with the tensor-core engine and with the NTT
engine, for N = 2^24, K = 4096 and T templates; one JSON line per case.
usage: python scripts/f3_bench.py [T ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402

N, K = 2 ** 24, 4096
Ts = [int(v) for v in sys.argv[1:]] or [148, 1024, 4096]
for engine in ("auto", "ntt"):
    plan = tm.Plan(N, K, seed=35, engine=engine)
    x, _, _ = plan.generate(0, 1, 0.0)
    y1, y2 = plan.fold(x)
    for T in Ts:
        _, t, _ = plan.generate(1, T, 0.1, want_x=False)
        ws = plan.workspace(T)
        for _ in range(3):
            plan.correlate_many(y1[0], y2[0], t, ws=ws)
        torch.cuda.synchronize()
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            plan.correlate_many(y1[0], y2[0], t, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        macs = T * 2 * (plan.M1 + 1) * K   # correlation MACs per call (both moduli, direct form)
        print(json.dumps({"engine": "tensor cores" if plan.corr_engine else "NTT", "N": N, "K": K, "templates": T,
                          "ms": round(ms, 4), "templates_per_s": round(T / ms * 1e3),
                          "effective_int8_TOPS": round(2 * macs / ms / 1e9, 1)}), flush=True)
