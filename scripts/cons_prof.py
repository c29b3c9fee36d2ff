"""Fold consumer profile of the fused kernel (variant built with -DTM_CONS_PROF):
cycles each consumer warp spent waiting for ring stages vs processing them."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, B = 2**20, 4096, 1024
plan = tm.Plan(N, K, seed=9)
x, t, _ = plan.generate(0, B, 0.1)
n = B * 8 + 4 * 148 + 24 * 148 + 64
dbg = torch.zeros(n, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    plan.run(x, t)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
d = dbg.cpu().numpy()[B * 8 + 4 * 148: B * 8 + 4 * 148 + 24 * 148].reshape(148, 8, 3)
w, b_, it_ = d[:, :, 0], d[:, :, 1], d[:, :, 2]
print('item-start waits (pempty/ydone) per CTA-warp p50 %.0f cycles = %.0f per item' % (np.median(it_), np.median(it_) / 7))
print('wait cycles per CTA-warp: p50 %.0f  busy: p50 %.0f  (busy share %.2f)' % (np.median(w), np.median(b_), np.median(b_ / (w + b_))))
print('per stage (1 MiB pair = 32 stages of 8 rows x 4096): wait %.0f busy %.0f cycles' % (np.median(w) / (7 * 32), np.median(b_) / (7 * 32)))
