import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, B = 2**20, 4096, 1024
plan = tm.Plan(N, K, seed=9)
x, t, _ = plan.generate(0, B, 0.1)
y1, y2 = plan.fold(x)
dbg = torch.zeros(B * 8 + 512, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    if len(sys.argv) > 1 and sys.argv[1] == 'run':
        plan.run(x, t)
    else:
        plan.correlate_match(y1, y2, t)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
dd = dbg.cpu().numpy()
d = dd[:B*8].reshape(B, 8)

ph = np.diff(d[:, :6], axis=1)
names = ['tmpl', 'stage_y', 'buildA', 'mma', 'epi']
for i, n in enumerate(names):
    print(f'{n:8s} mean {ph[:, i].mean():9.0f} p50 {np.median(ph[:, i]):9.0f} max {ph[:, i].max():9.0f}')
last = ph[B - 148:]  # each CTA's last pair (static schedule)
print('last pairs: ' + '  '.join(f'{n} {np.median(last[:, i]):.0f}' for i, n in enumerate(names)))
tot = d[:, 5] - d[:, 0]
print('pair lifetime mean', tot.mean(), 'span per SM', [(d[d[:,6]==s,5].max()-d[d[:,6]==s,0].min()) for s in range(3)])
t0 = d[:, 0].min()
sms = np.unique(d[:, 6])
first = np.array([d[d[:, 6] == s, 0].min() - t0 for s in sms]) / 1e3
last = np.array([d[d[:, 6] == s, 5].max() - t0 for s in sms]) / 1e3
print('(ns stamps) first TC start per SM us: min %.1f p50 %.1f max %.1f' % (first.min(), np.median(first), first.max()))
print('last TC end per SM us: min %.1f p50 %.1f max %.1f' % (last.min(), np.median(last), last.max()))
cnt = np.array([(d[:, 6] == s).sum() for s in sms])
print('pairs per SM', np.bincount(cnt))
if len(sys.argv) > 1 and sys.argv[1] == 'run':
    ex = dd[B * 8: B * 8 + 296].reshape(148, 2)
    k0 = ex[:, 0].min()
    print('CTA entry us: max %.1f; TC exit us: min %.1f p50 %.1f max %.1f' % ((ex[:, 0].max() - k0) / 1e3, (ex[:, 1].min() - k0) / 1e3, np.median(ex[:, 1] - k0) / 1e3, (ex[:, 1].max() - k0) / 1e3))
    fe = dd[B * 8 + 296: B * 8 + 296 + 148]
    tail = ex[:, 1] - fe
    print('last fold item end us: min %.1f p50 %.1f max %.1f; TC tail after it us: min %.1f p50 %.1f max %.1f' % ((fe.min() - k0) / 1e3, (np.median(fe) - k0) / 1e3, (fe.max() - k0) / 1e3, tail.min() / 1e3, np.median(tail) / 1e3, tail.max() / 1e3))
    ep = dd[B * 8 + 444: B * 8 + 444 + 148]
    print('fold epilogue (last item) us: min %.1f p50 %.1f max %.1f' % (ep.min() / 1e3, np.median(ep) / 1e3, ep.max() / 1e3))
    print('first TC start after kernel entry us: min %.1f p50 %.1f max %.1f' % ((first.min()*1e3 + t0 - k0) / 1e3, (np.median(first)*1e3 + t0 - k0) / 1e3, (first.max()*1e3 + t0 - k0) / 1e3))
