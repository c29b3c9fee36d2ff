"""Per-CTA phase timeline of corr_tc_tiled (instrumented via tm_debug_tc_timestamps).
usage: python scripts/tiled_phases.py N K B"""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, '.')
os.environ['TM_TC_TILED'] = '1'
import paper_1509_04863_b200 as tm
L = tm.lib()
N, K, B = (int(v) for v in sys.argv[1:4])
plan = tm.Plan(N, K, seed=9)
x, t, _ = plan.generate(0, B, 0.1)
y1, y2 = plan.fold(x)
nmax = 1 << 16
dbg = torch.zeros(nmax * 8, dtype=torch.int64, device='cuda')
L.tm_debug_tc_timestamps.argtypes = [ctypes.c_void_p]
for it in range(3):
    L.tm_debug_tc_timestamps(dbg.data_ptr() if it == 2 else None)
    if it == 2:
        dbg.zero_()
    plan.correlate_match(y1, y2, t)
torch.cuda.synchronize()
L.tm_debug_tc_timestamps(None)
d = dbg.cpu().numpy().reshape(nmax, 8)
d = d[d[:, 0] != 0]
t0 = d[:, 0].min()
sm = d[:, 7] >> 32
passes = (d[:, 7] >> 8) & 0xFFFF
nsp = (d[:, 7] >> 24) & 0xFF
nl = d[:, 7] & 0xFF
print(f'CTAs {len(d)}, SMs {len(np.unique(sm))}, passes p50 {np.median(passes)}, nl {np.bincount(nl)}')
for name, v in [('start', d[:, 0] - t0), ('scan+alloc', d[:, 1] - d[:, 0]), ('loop', d[:, 2] - d[:, 1]),
                ('epilogue', d[:, 3] - d[:, 2]), ('end', d[:, 3] - t0),
                ('epi: 1st TMEM ld', np.where(d[:, 5] > 0, d[:, 5] - d[:, 2], 0)),
                ('epi: outputs done', np.where(d[:, 6] > 0, d[:, 6] - d[:, 2], 0)),
                ('arrive+finish', np.where(d[:, 4] > 0, d[:, 4] - d[:, 3], 0)),
                ('exit', np.where(d[:, 4] > 0, d[:, 4] - t0, 0))]:
    v = v / 1e3
    print(f'{name:14s} us: min {v.min():7.2f} p50 {np.median(v):7.2f} max {v.max():7.2f}')
epi = (d[:, 3] - d[:, 2]) / 1e3
for lo, hi in [(0, 0), (1, 4), (5, 9), (10, 14), (15, 19), (20, 24)]:
    m = (nsp >= lo) & (nsp <= hi)
    if m.any():
        print(f'nsp {lo:2d}..{hi:2d}: {m.sum():4d} CTAs, epilogue us p50 {np.median(epi[m]):6.2f} max {epi[m].max():6.2f}')
