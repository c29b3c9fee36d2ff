"""Success rate against the planted shift across K at N = 2^31 (cfg5's signal) and
N = 2^24 (cfg4), through tm_run on device-generated pairs: the K^2 / log K >= O(N)
transition of PAPER.md P:360-362 (SURVEY 8(d) companions).  Prints one JSON line.

    python scripts/k_transition.py [pairs_cfg5] [pairs_cfg4]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402


def rate(N, K, pairs, noise, seed, batch):
    plan = tm.Plan(N, K, seed=seed, inputs_stable=True)
    ok, ks, ms = 0, [], []
    for p0 in range(0, pairs, batch):
        b = min(batch, pairs - p0)
        x, t, k0 = plan.generate(p0, b, noise)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res, k = plan.run(x, t)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1) / b)
        ok += int((k == k0).sum())
        ks += [(int(a), int(c)) for a, c in zip(k.tolist(), k0.tolist())]
        del x, t
    return {"N": N, "K": K, "pairs": pairs, "noise": noise, "success": ok / pairs,
            "ms_per_pair_first_call": ms[0], "ms_per_pair_median": sorted(ms)[len(ms) // 2],
            "engine": "tensor cores" if plan.corr_engine else "ntt", "path": tm.RUN_PATHS[plan.run_path(batch)],
            "k_vs_k0": ks[:8]}


def main():
    p5 = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    p4 = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    out = {"what": "success rate vs K (P:360-362); tm_run on device-generated pairs (tmgen recipe)", "rows": []}
    t0 = time.time()
    for K in (65536, 2 ** 18, 2 ** 19):
        out["rows"].append(rate(2 ** 31, K, p5, 0.05, 5, 1))
    for K in (4096, 8192, 16384, 32768, 65536):
        out["rows"].append(rate(2 ** 24, K, p4, 0.2, 4, 64))
    out["seconds"] = time.time() - t0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
