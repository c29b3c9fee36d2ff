import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, B = 2**20, 4096, 1024
plan = tm.Plan(N, K, seed=9)
x, t, _ = plan.generate(0, B, 0.1)
y1, y2 = plan.fold(x)
dbg = torch.zeros(B * 8 + 256, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    plan.correlate_match(y1, y2, t)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
dd = dbg.cpu().numpy()
d = dd[:B*8].reshape(B, 8)

ph = np.diff(d[:, :6], axis=1)
names = ['tmpl', 'stage_y', 'buildA', 'mma', 'epi']
for i, n in enumerate(names):
    print(f'{n:8s} mean {ph[:, i].mean():9.0f} p50 {np.median(ph[:, i]):9.0f} max {ph[:, i].max():9.0f}')
tot = d[:, 5] - d[:, 0]
print('cta lifetime mean', tot.mean(), 'span per SM', [(d[d[:,6]==s,5].max()-d[d[:,6]==s,0].min()) for s in range(3)])
