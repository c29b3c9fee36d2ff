"""The README usage example as a runnable check (staged path == fused path)."""
import sys; sys.path.insert(0, '/root/repo')
import paper_1509_04863_b200 as tm
plan = tm.Plan(N=2**20, K=4096, seed=2)                 # Alg. 1 step 2: M1 = K, M2 = K + 1
x, t, k0 = plan.generate(0, 1024, 0.1)                  # seeded synthetic +-1 pairs, planted shifts
residues, k = plan.run(x, t)                            # steps 3-9 in one fused kernel; k = -1: no match
y1, y2 = plan.fold(x)                                   # or stage by stage:
r1, r2 = plan.correlate(y1, y2, plan.fold_template(t))
residues2, k2 = plan.match(r1, r2)
import torch
assert torch.equal(k, k2) and torch.equal(residues, residues2)
print("readme snippet ok", float((k == k0).double().mean()))
