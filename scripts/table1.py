"""Reproduce PAPER.md Table 1 with the CUDA path: K = N/2^10,
noiseless +-1 codes, M1 = K, M2 = K+1, 1000 trials per column (the paper's
count), device-generated trials.  Writes one JSON object to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402

PAPER = {23: 0.05, 24: 0.21, 25: 0.85, 26: 1.0, 27: 1.0}
trials = int(os.environ.get("TRIALS", "1000"))
out = {"table": "PAPER.md Table 1, K = N/2^10", "trials": trials, "rows": []}
for logN, p in PAPER.items():
    N = 2 ** logN
    plan = tm.Plan(N, N >> 10, seed=1509)
    B = max(1, min(trials, (1 << 31) // N))
    ok = done = 0
    t0 = time.time()
    while done < trials:
        nb = min(B, trials - done)
        x, t, k0 = plan.generate(done, nb, 0.0)
        _, k = plan.run(x, t)
        ok += int((k == k0).sum())
        done += nb
    torch.cuda.synchronize()
    out["rows"].append({"log2N": logN, "K": N >> 10, "success": ok / trials, "paper": p,
                        "seconds": round(time.time() - t0, 2)})
print(json.dumps(out))
