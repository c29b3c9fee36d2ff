"""Feasibility probe (A/B only): the batch split into chunks, the fold of chunk
c+1 (caller stream) concurrent with the tiled correlation of chunk c (side
stream), vs the staged sequence.  Run with TM_LIB_VARIANT=cores (smaller fold
ring and item rows, tiled kernel at <= 68 registers) so that one CTA of each
kernel can share an SM.  usage: python scripts/overlap_probe.py N K B chunks"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402

os.environ.setdefault("TM_TC_TILED", "1")
N, K, B, C = (int(v) for v in sys.argv[1:5])
plan = tm.Plan(N, K, seed=4, inputs_stable=True)
x, t, k0 = plan.generate(0, B, 0.2)
per = B // C
ws_f = [plan.workspace(per) for _ in range(C)]
ws_c = [plan.workspace(per) for _ in range(C)]
y1 = torch.empty((B, plan.len_y1), dtype=torch.int32, device="cuda")
y2 = torch.empty((B, plan.len_y2), dtype=torch.int32, device="cuda")
res = torch.empty((B, 2), dtype=torch.int32, device="cuda")
k = torch.empty(B, dtype=torch.int64, device="cuda")
s0 = torch.cuda.current_stream()
s1 = torch.cuda.Stream()
ev = [torch.cuda.Event() for _ in range(C)]


def staged():
    plan.run(x, t, residues=res, k=k, ws=ws_f[0] if C == 1 else plan_ws)


plan_ws = plan.workspace(B)


def chunked():
    for c in range(C):
        sl = slice(c * per, (c + 1) * per)
        plan.fold(x[sl], y1=y1[sl], y2=y2[sl], ws=ws_f[c], stream=s0)
        ev[c].record(s0)
        s1.wait_event(ev[c])
        plan.correlate_match(y1[sl], y2[sl], t[sl], residues=res[sl], k=k[sl], ws=ws_c[c], stream=s1)
    done = torch.cuda.Event()
    done.record(s1)
    s0.wait_event(done)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(reps):
        fn()
    b.record(s0)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_staged = timeit(lambda: plan.run(x, t, residues=res, k=k, ws=plan_ws))
k_ref = k.clone()
t_chunk = timeit(chunked)
same = bool(torch.equal(k, k_ref))
print(f"N={N} K={K} B={B} chunks={C} variant={os.environ.get('TM_LIB_VARIANT', 'base')}: "
      f"staged {t_staged:.4f} ms, chunked+overlap {t_chunk:.4f} ms, same k {same}")
