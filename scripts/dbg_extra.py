import os, sys
sys.path.insert(0, '/root/repo'); os.chdir('/root/repo')
import numpy as np, torch
import oracle
import paper_1509_04863_b200 as tm
N, K, M1, nparts = 167073, 661, 2304, 7
rng = np.random.default_rng(5)
B = 2
plan = tm.Plan(N, K, M=M1, seed=7, binary=False)
print("engine", plan.corr_engine, "M1 M2", plan.M1, plan.M2)
x_h = rng.integers(-8, 9, (B, N)).astype(np.int8)
k0 = rng.integers(0, N, B)
t_h = np.stack([x_h[b][(k0[b] + np.arange(K)) % N] for b in range(B)]).astype(np.int8)
x, t = torch.from_numpy(x_h).cuda(), torch.from_numpy(t_h).cuda()
y1, y2 = plan.fold(x)
r1, r2 = plan.correlate(y1, y2, plan.fold_template(t))
res_s, k_s = plan.match(r1, r2)
res_w, k_w = plan.correlate_match(y1, y2, t)
res_r, k_r = plan.run(x, t)
torch.cuda.synchronize()
for np_ in (1, 2, 7):
    keys = None
    allk = []
    for part in range(np_):
        kp = plan.correlate_match_part(y1, y2, t, part, np_)
        torch.cuda.synchronize()
        allk.append(kp.cpu().numpy().copy())
        keys = kp.clone() if keys is None else torch.maximum(keys, kp)
    res, k = plan.match_keys(keys)
    torch.cuda.synchronize()
    print("nparts", np_, "res", res.cpu().numpy().tolist(), "k", k.cpu().numpy().tolist())
    if np_ == 7:
        for part, kk in enumerate(allk):
            print("   part", part, [hex(int(v) & (2**64 - 1)) for v in kk.ravel()])
for b in range(B):
    o = oracle.ftm(x_h[b], t_h[b], M=M1)
    print("pair", b, "oracle", o["residues"], o["k"], "staged", res_s[b].tolist(), int(k_s[b]), "whole", res_w[b].tolist(), int(k_w[b]), "run", res_r[b].tolist(), int(k_r[b]),
          "y ok", np.array_equal(y1[b].cpu().numpy(), o["y1"]), np.array_equal(y2[b].cpu().numpy(), o["y2"]),
          "r ok", np.array_equal(r1[b].cpu().numpy(), o["r1"]), np.array_equal(r2[b].cpu().numpy(), o["r2"]))
    r2o = o["r2"]; print("   oracle r2 max", int(r2o.max()), "at", int(np.argmax(r2o)), "r2[M1]", int(r2o[M1]), "r1 max", int(o["r1"].max()), int(np.argmax(o["r1"])))
