"""Debug: one sweep_wide seed, where r differs from the oracle (indices, differences)."""
import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); os.chdir('/root/repo')
import importlib.util
import numpy as np, torch
spec = importlib.util.spec_from_file_location("sw", "/root/repo/scripts/sweep_wide.py")
import oracle
import paper_1509_04863_b200 as tm
seed = int(sys.argv[1])
# sweep_wide's case()
def case(rng):
    dtype = "float32" if rng.random() < 0.2 else "int8"
    K = int(rng.integers(1, 6000))
    M = 0 if rng.random() < 0.6 else int(K + rng.integers(0, 3000))
    M1 = max(M or K, 2)
    if M == 0 and K < 2:
        M = 2
    N = int(rng.integers(max(K, 2), min(M1 * (M1 + 1) - 1, 1 << 22) + 1))
    if rng.random() < 0.5:
        N = max(M1, (N // M1) * M1)
    binary = dtype == "int8" and rng.random() < 0.7
    block = rng.random() < 0.2
    alias = (not block) and N % M1 == 0 and rng.random() < 0.2
    engine = rng.choice(["auto", "ntt"]) if dtype == "int8" else None
    return N, K, M, dtype, binary, block, alias, engine
rng = np.random.default_rng(1000 + seed)
N, K, M, dtype, binary, block, alias, engine = case(rng)
B = int(rng.integers(1, 4))
print("case", N, K, M, dtype, binary, block, alias, engine, "B", B)
plan = tm.Plan(N, K, M=M, seed=seed, dtype=dtype, binary=binary, engine=engine, block=block, alias_repair=alias)
x_h = (1 - 2 * rng.integers(0, 2, (B, N))).astype(np.int8) if binary else rng.integers(-128, 128, (B, N)).astype(np.int8)
k0 = rng.integers(0, N, B)
t_h = np.stack([x_h[b][(k0[b] + np.arange(K)) % N] for b in range(B)]).astype(np.int8)
x, t = torch.from_numpy(x_h).cuda(), torch.from_numpy(t_h).cuda()
for rep in range(2):
    y1, y2 = plan.fold(x)
    tf = plan.fold_template(t)
    r1, r2 = plan.correlate(y1, y2, tf)
    torch.cuda.synchronize()
    for b in range(B):
        o = oracle.ftm(x_h[b], t_h[b], M=plan.M1 if plan.M1 != plan.K else 0)
        print("rep", rep, "pair", b, "y ok", np.array_equal(y1[b].cpu().numpy(), o["y1"]), np.array_equal(y2[b].cpu().numpy(), o["y2"]),
              "max|y2|", int(np.abs(o["y2"]).max()))
        for name, g, ref in (("r1", r1, o["r1"]), ("r2", r2, o["r2"])):
            d = g[b].cpu().numpy() - ref
            bad = np.nonzero(d)[0]
            print("  ", name, "mismatch", len(bad), "idx", bad[:6], "..", bad[-3:], "diff", d[bad[:4]])
        # is the r2 difference a sum over a tail of y2?  r2[k] = sum_i t[i] y2[k+i]
        d = r2[b].cpu().numpy() - o["r2"]
        bad = np.nonzero(d)[0]
        if len(bad):
            kk = int(bad[0]); y = o["y2"].astype(np.int64); tt = t_h[b].astype(np.int64)
            terms = tt * y[kk:kk + K]
            cs = np.cumsum(terms[::-1])[::-1]   # suffix sums: terms i >= j
            hit = np.nonzero(cs == -d[kk])[0]
            print("   r2[%d] diff %d = minus suffix of terms from i =" % (kk, d[kk]), hit[:5], " (K=%d, y idx %s)" % (K, (kk + hit[:5])))
            for CR in (8, 11, 16, 17, 32):
                for kk2 in (0, 1, 66):
                    terms2 = tt * y[kk2:kk2 + K]
                    idx = kk2 + np.arange(K)
                    parts = [int(terms2[(idx >= 128 * c0) & (idx < 128 * (c0 + CR))].sum()) for c0 in range(0, 64, CR)]
                    m = [i for i, v in enumerate(parts) if v == -d[kk2] or v == d[kk2]]
                    if m:
                        print("   CR", CR, "k", kk2, "diff", d[kk2], "= +-range partial", m, parts[m[0]])
            pre = np.cumsum(terms); hit2 = np.nonzero(pre == -d[kk])[0]; print("   or minus prefix up to i =", hit2[:5])
