"""Two-stream step pipelining (paper_1509_04863_b200/pipeline.py, SingleSignal(depth=)):
consecutive steps over DIFFERENT inputs, the fold of step i+1 concurrent with the
correlation of step i.  Every step's residues and k must equal the one-stream
tm_run's and the oracle's Algorithm 1 -- a buffer set reused too
early, or a result read from the wrong slot, shows up as another step's answer."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tm():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1509_04863_b200 as tm
    return tm


@pytest.mark.parametrize("N,K,B,dtype,depth", [
    (1 << 21, 8192, 6, "int8", 2),      # staged: split-item fold + tiled tensor-core correlation
    (1 << 21, 8192, 6, "int8", 3),
    (1 << 18, 2048, 5, "float32", 2),   # staged: fp32 strips + FFT correlation
    (1 << 16, 1024, 7, "int8", 2),      # fused one-kernel path: run as is
])
def test_pipeline_steps_equal_run_and_oracle(tm, N, K, B, dtype, depth):
    plan = tm.Plan(N, K, seed=11, dtype=dtype)
    pipe = tm.Pipeline(plan, B, depth=depth)
    steps = 2 * depth + 1
    inputs = [plan.generate(100 * i, B, 0.05) for i in range(steps)]
    got = []
    for x, t, _ in inputs:
        res, k = pipe.step(x, t)
        pipe.drain()
        got.append((res.clone(), k.clone()))   # (cloned on the current stream, after the drain)
    # the same steps back to back without draining in between: slots rotate under overlap
    keep = []
    for i, (x, t, _) in enumerate(inputs):
        res, k = pipe.step(x, t)
        if i >= steps - depth:                 # the last `depth` results are still in their slots
            keep.append((i, res, k))
    pipe.drain()
    torch.cuda.synchronize()
    for i, (x, t, _) in enumerate(inputs):
        r_ref, k_ref = plan.run(x, t)
        torch.cuda.synchronize()
        assert torch.equal(got[i][1], k_ref) and torch.equal(got[i][0], r_ref), i
    for i, res, k in keep:
        assert torch.equal(k, got[i][1]) and torch.equal(res, got[i][0]), i
    if dtype == "int8":
        x, t, _ = inputs[-1]
        xh, th = x.cpu().numpy(), t.cpu().numpy()
        for b in (0, B - 1):
            o = oracle.ftm(xh[b], th[b])
            assert tuple(got[-1][0][b].tolist()) == o["residues"] and int(got[-1][1][b]) == o["k"]


@pytest.mark.parametrize("depth", [2, 3])
def test_single_signal_depth_equals_one_stream_and_oracle(tm, depth):
    from paper_1509_04863_b200.single import SingleSignal
    N, K = 1 << 24, 8192
    plan = tm.Plan(N, K, seed=5)
    ss1 = SingleSignal(plan, 0, 1)
    ssd = SingleSignal(plan, 0, 1, depth=depth)
    sigs = [plan.generate(i, 1, 0.05) for i in range(2 * depth + 1)]
    outs = []
    for x, t, _ in sigs:
        res, k = ssd.step(x, t)
        outs.append((res, k, ssd.y1, ssd.y2))
        if len(outs) % depth == 0 or len(outs) == len(sigs):   # check before the slots are reused
            ssd.drain()
            torch.cuda.synchronize()
            n = len(outs)
            for j in range(max(0, n - depth), n):
                xs, ts, _ = sigs[j]
                r1, k1 = ss1.step(xs, ts)
                torch.cuda.synchronize()
                assert torch.equal(outs[j][1], k1) and torch.equal(outs[j][0], r1), j
                assert torch.equal(outs[j][2], ss1.y1) and torch.equal(outs[j][3], ss1.y2), j
    x, t, _ = sigs[-1]
    o = oracle.ftm(x[0].cpu().numpy(), t[0].cpu().numpy())
    assert tuple(outs[-1][0][0].tolist()) == o["residues"] and int(outs[-1][1][0]) == o["k"]
    assert np.array_equal(outs[-1][2][0].cpu().numpy(), o["y1"])
    assert np.array_equal(outs[-1][3][0].cpu().numpy(), o["y2"])
