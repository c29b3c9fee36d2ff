"""A/B probe: consecutive steps software-pipelined over two streams -- the fold of
step i+1 (caller stream) concurrent with the correlation + match of step i (side
stream, double-buffered y / workspace / results) -- against back-to-back tm_run.
usage: python scripts/pipeline_probe.py N K B int8|float32 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_04863_b200 as tm  # noqa: E402

N, K, B = (int(v) for v in sys.argv[1:4])
dtype = sys.argv[4] if len(sys.argv) > 4 else "int8"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
plan = tm.Plan(N, K, seed=4, dtype=dtype, inputs_stable=True)
x, t, k0 = plan.generate(0, B, 0.1)
ydt = plan.y_dtype
s0 = torch.cuda.current_stream()
ws_run = plan.workspace(B)
res = torch.empty((B, 2), dtype=torch.int32, device="cuda")
k = torch.empty(B, dtype=torch.int64, device="cuda")


def timeit(fn, after=None):
    for _ in range(5):
        fn()
    if after:
        after()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s0)
    for _ in range(reps):
        fn()
    if after:
        after()
    b.record(s0)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_run = timeit(lambda: plan.run(x, t, residues=res, k=k, ws=ws_run))
k_ref = k.clone()


def staged_one_stream():
    plan.fold(x, y1=Y1[0], y2=Y2[0], ws=WF[0], stream=s0)
    plan.correlate_match(Y1[0], Y2[0], t, residues=R[0], k=KK[0], ws=WC[0], stream=s0)


Y1 = [torch.empty((B, plan.len_y1), dtype=ydt, device="cuda") for _ in range(2)]
Y2 = [torch.empty((B, plan.len_y2), dtype=ydt, device="cuda") for _ in range(2)]
WF = [plan.workspace(B) for _ in range(2)]
WC = [plan.workspace(B) for _ in range(2)]
R = [torch.empty((B, 2), dtype=torch.int32, device="cuda") for _ in range(2)]
KK = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(2)]
t_st = timeit(staged_one_stream)
same_st = bool(torch.equal(KK[0], k_ref))

out = [f"N={N} K={K} B={B} {dtype}: tm_run {t_run:.4f} ms, fold+correlate_match one stream {t_st:.4f} (k same {same_st})"]
def variant(nbuf, fold_prio, corr_prio):
    global s0
    sf = torch.cuda.Stream(priority=fold_prio)
    s1 = torch.cuda.Stream(priority=corr_prio)
    while len(Y1) < nbuf:
        Y1.append(torch.empty_like(Y1[0])); Y2.append(torch.empty_like(Y2[0]))
        WF.append(plan.workspace(B)); WC.append(plan.workspace(B))
        R.append(torch.empty_like(R[0])); KK.append(torch.empty_like(KK[0]))
    folded = [torch.cuda.Event() for _ in range(nbuf)]
    done = [torch.cuda.Event() for _ in range(nbuf)]
    state = {"i": 0}
    for d in done:
        d.record(s1)

    def step():
        b = state["i"] % nbuf
        state["i"] += 1
        sf.wait_event(done[b])  # buffers b are free once step i-nbuf's correlation has read them
        plan.fold(x, y1=Y1[b], y2=Y2[b], ws=WF[b], stream=sf)
        folded[b].record(sf)
        s1.wait_event(folded[b])
        plan.correlate_match(Y1[b], Y2[b], t, residues=R[b], k=KK[b], ws=WC[b], stream=s1)
        done[b].record(s1)

    def drain():
        for d in done:
            s0.wait_event(d)

    for kk in KK:
        kk.fill_(-7)
    sf.wait_stream(s0)
    t_p = timeit(step, drain)
    same = all(bool(torch.equal(kk, k_ref)) for kk in KK[:nbuf])
    out.append(f"pipelined nbuf {nbuf} fold prio {fold_prio} corr prio {corr_prio}: {t_p:.4f} ms (k same {same})")


for nb, fp, cp in ((2, 0, 0), (3, 0, 0), (2, -1, 0), (3, -1, 0), (2, 0, -1)):
    variant(nb, fp, cp)
print("\n  ".join(out), flush=True)
