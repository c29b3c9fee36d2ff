import sys, os; sys.path.insert(0, '/root/repo')
import torch, paper_1509_04863_b200 as tm
N, K = 2 ** 20, 4096
for B in (16, 32, 64, 100, 148, 296):
    plan = tm.Plan(N, K, seed=5)
    x, t, _ = plan.generate(0, B, 0.1)
    ws = plan.workspace(B)
    for _ in range(5): plan.run(x, t, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): plan.run(x, t, ws=ws)
    e1.record(); torch.cuda.synchronize()
    print(os.environ.get("TM_FUSED_TC", "1"), B, plan.run_path(B), round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
