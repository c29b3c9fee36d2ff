"""Randomized parity sweep of the alpha-modulus plans (tm_mplan) and the split
correlation (tm_correlate_match_part) against the oracle (not part of pytest).
usage: python scripts/sweep_extra.py n_cases"""
import math
import os
import sys

sys.path.insert(0, '/root/repo')
os.chdir('/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1509_04863_b200 as tm  # noqa: E402

n = int(sys.argv[1])
rng = np.random.default_rng(2026)
fails = 0
for c in range(n):
    try:
        if c % 2 == 0:   # alpha moduli
            K = int(rng.integers(2, 200))
            alpha = int(rng.integers(2, 5))
            M = []
            cand = K + int(rng.integers(0, 50))
            while len(M) < alpha:
                if all(math.gcd(cand, m) == 1 for m in M):
                    M.append(cand)
                cand += 1
            P = int(np.prod(M))
            N = int(rng.integers(K + 1, min(P, 200000)))
            B = int(rng.integers(1, 4))
            binary = rng.random() < 0.5
            plan = tm.MultiPlan(N, K, M, binary=binary)
            if binary:
                x_h = (1 - 2 * rng.integers(0, 2, (B, N))).astype(np.int8)
            else:
                x_h = rng.integers(-128, 128, (B, N)).astype(np.int8)
            k0 = rng.integers(0, N, B)
            t_h = np.stack([x_h[b][(k0[b] + np.arange(K)) % N] for b in range(B)]).astype(np.int8)
            res, k = plan.run(torch.from_numpy(x_h).cuda(), torch.from_numpy(t_h).cuda())
            res, k = res.cpu().numpy(), k.cpu().numpy()
            for b in range(B):
                o = oracle.ftm_multi(x_h[b], t_h[b], M)
                assert tuple(int(v) for v in res[b]) == o["residues"] and int(k[b]) == o["k"], (c, N, K, M, b)
        else:            # split correlation
            M1 = 128 * int(rng.integers(1, 80))
            K = int(rng.integers(1, M1 + 1))
            q = int(rng.integers(2, 200))
            N = M1 * q if rng.random() < 0.7 else M1 * q - int(rng.integers(1, M1))
            if M1 * (M1 + 1) <= N:
                continue
            B = int(rng.integers(1, 3))
            plan = tm.Plan(N, K, M=M1 if M1 != K else 0, seed=c, binary=False)
            x_h = rng.integers(-8, 9, (B, N)).astype(np.int8)
            k0 = rng.integers(0, N, B)
            t_h = np.stack([x_h[b][(k0[b] + np.arange(K)) % N] for b in range(B)]).astype(np.int8)
            x, t = torch.from_numpy(x_h).cuda(), torch.from_numpy(t_h).cuda()
            y1, y2 = plan.fold(x)
            nparts = int(rng.integers(1, 9))
            keys = None
            for part in range(nparts):
                kp = plan.correlate_match_part(y1, y2, t, part, nparts)
                keys = kp.clone() if keys is None else torch.maximum(keys, kp)
            res, k = plan.match_keys(keys)
            res, k = res.cpu().numpy(), k.cpu().numpy()
            for b in range(B):
                o = oracle.ftm(x_h[b], t_h[b], M=M1 if M1 != K else 0, want_vectors=False)
                assert tuple(int(v) for v in res[b]) == o["residues"] and int(k[b]) == o["k"], (c, N, K, M1, nparts, b)
    except tm.TMError as e:
        if "not eligible" in str(e) or "EUNSUPPORTED" in str(e):
            continue
        fails += 1
        print("FAIL", c, repr(e)[:300], flush=True)
    except Exception as e:
        fails += 1
        print("FAIL", c, repr(e)[:300], flush=True)
        if "CUDA error" in repr(e):
            break
print("done", n, "fails", fails)
