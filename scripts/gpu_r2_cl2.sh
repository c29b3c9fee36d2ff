TM_DEBUG_CL=1 python - <<'PY'
import torch, paper_1509_04863_b200 as tm
for N,K,B in [(2**31, 65536, 1), (2**20, 8192, 2), (2**24, 16384, 4)]:
    plan = tm.Plan(N, K, seed=1)
    x, t, _ = plan.generate(0, B, 0.05)
    plan.run(x, t); torch.cuda.synchronize(); print(N, K, B, "ok", flush=True)
    del x, t
PY
