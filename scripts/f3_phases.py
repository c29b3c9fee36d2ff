import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, T = 2**24, 4096, 1024
plan = tm.Plan(N, K, seed=9)
x, _, _ = plan.generate(0, 1, 0.0)
y1, y2 = plan.fold(x)
_, t, _ = plan.generate(1, T, 0.1, want_x=False)
dbg = torch.zeros(T * 8 + 512, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
ws = plan.workspace(T)
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    plan.correlate_many(y1[0], y2[0], t, ws=ws)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
d = dbg.cpu().numpy()[:T*8].reshape(T, 8)
ph = np.diff(d[:, :6], axis=1)
for i, n in enumerate(['tmpl', 'stage_y', 'buildA', 'mma', 'epi']):
    print(f'{n:8s} mean {ph[:, i].mean():9.0f} p50 {np.median(ph[:, i]):9.0f} max {ph[:, i].max():9.0f}')
print('lifetime mean', (d[:,5]-d[:,0]).mean(), 'span', (d[:,5].max()-d[:,0].min()))
