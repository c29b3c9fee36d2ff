"""Owner-epilogue phase times of the fused kernel's last pair per CTA (variant -DTM_EPI_PROF)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, B = 2**20, 4096, 1024
plan = tm.Plan(N, K, seed=9)
x, t, _ = plan.generate(0, B, 0.1)
n = B * 8 + 8 * 148 + 64
dbg = torch.zeros(n, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    plan.run(x, t)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
d = dbg.cpu().numpy()[B * 8 + 4 * 148: B * 8 + 8 * 148].reshape(148, 4) / 1e3
print('epilogue us (from pfull): p50 stamps', [round(float(np.median(d[:, i])), 2) for i in range(4)])
