import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_1509_04863_b200 as tm, oracle, tmgen
N, K = 2 ** 20, 4096
for B in (4096, 149, 296, 1):
    plan = tm.Plan(N, K, seed=5)
    x, t, k0 = plan.generate(0, B, 0.1)
    res, k = plan.run(x, t)
    torch.cuda.synchronize()
    rr, kk = res.cpu().numpy(), k.cpu().numpy()
    bad = 0
    for b in sorted(set([0, B // 3, B // 2, B - 1])):
        xb = tmgen.signal(5, b, N); tb = tmgen.template(5, b, N, K, 0.1)
        o = oracle.ftm(xb, tb, want_vectors=False)
        bad += (tuple(rr[b]) != o["residues"]) or (kk[b] != o["k"])
    print(B, plan.run_path(B), "mismatches", bad, "success", float((k == k0).double().mean()))
