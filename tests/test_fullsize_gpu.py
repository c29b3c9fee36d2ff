"""Parity at BASELINE.json's full sizes: EVERY pair of cfg2, cfg3
and cfg4 (each K of the sweep), and the whole cfg5 signal, compared with the CPU
oracle (one oracle process per host core, tests/oracle_pool.py); the extreme
inputs of the integer path (all-ones cfg5: y = 2^15, r = 2^31; all +127 general
int8 data: 4-bit limbs 0..3 of the tiled tensor-core engine); and the fused
kernel's own y rows (plan flag TM_KEEP_Y) against the staged fold, every pair.
Inputs come from the host generator (tmgen) and are uploaded; expected values
come only from oracle/ or from closed forms stated in the test.
"""
import numpy as np
import pytest

import oracle
import tmgen
from oracle_pool import ftm_pairs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda:0"


@pytest.fixture(scope="module")
def tm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04863_b200 import _build
    _build.build()
    import paper_1509_04863_b200 as m
    return m


def up(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def staged_and_run(plan, x, t):
    """fold -> fold_template -> correlate -> match (staged) and tm_run on the same batch."""
    y1, y2 = plan.fold(x)
    r1, r2 = plan.correlate(y1, y2, plan.fold_template(t))
    res, k = plan.match(r1, r2)
    res_run, k_run = plan.run(x, t)
    torch.cuda.synchronize()
    return [v.cpu().numpy() for v in (y1, y2, r1, r2, res, k, res_run, k_run)]


@pytest.mark.parametrize("cfg", ["cfg2", "cfg4a", "cfg4b", "cfg4"])
def test_every_pair_int(tm, cfg):
    """Integer configs, every pair: y1, y2, r1, r2 (staged kernels), residues and
    k (staged and tm_run -- the fused kernel at cfg2, fold + correlation kernels
    at cfg4) byte-identical to the oracle."""
    N, K, B, noise, seed = {"cfg2": (2 ** 20, 4096, 1024, 0.1, 2), "cfg4a": (2 ** 24, 4096, 64, 0.2, 4),
                            "cfg4b": (2 ** 24, 8192, 64, 0.2, 4), "cfg4": (2 ** 24, 16384, 64, 0.2, 4)}[cfg]
    plan = tm.Plan(N, K, seed=seed)
    x_h, t_h, k0 = tmgen.batch(seed, 0, B, N, K, noise)
    y1, y2, r1, r2, res, k, res_run, k_run = staged_and_run(plan, up(x_h), up(t_h))
    del x_h
    orc = ftm_pairs(seed, range(B), N, K, noise)
    for b, o in enumerate(orc):
        assert o["pair"] == b
        np.testing.assert_array_equal(y1[b], o["y1"], err_msg=f"{cfg} y1 pair {b}")
        np.testing.assert_array_equal(y2[b], o["y2"], err_msg=f"{cfg} y2 pair {b}")
        np.testing.assert_array_equal(r1[b], o["r1"], err_msg=f"{cfg} r1 pair {b}")
        np.testing.assert_array_equal(r2[b], o["r2"], err_msg=f"{cfg} r2 pair {b}")
        assert tuple(res[b]) == o["residues"] == tuple(res_run[b]), (cfg, b)
        assert k[b] == o["k"] == k_run[b], (cfg, b)
    print(f"{cfg}: {B} pairs identical to the oracle; success rate {np.mean(k_run == k0):.3f}")


def test_every_pair_cfg3_fp32(tm):
    """cfg3 (fp32, N = 2^22, K = 8192, 256 pairs), every pair, reading C15: y and r
    within 1e-5 of max |oracle| per vector, residues identical unless the oracle's
    top-two gap is within that bound, k = CRT(GPU residues) and equal to the
    oracle's whenever the residues are."""
    N, K, B, noise, seed = 2 ** 22, 8192, 256, 0.5, 3
    plan = tm.Plan(N, K, seed=seed, dtype="float32")
    x_h, t_h, k0 = tmgen.batch(seed, 0, B, N, K, noise, dtype=np.float32)
    y1, y2, r1, r2, res, k, res_run, k_run = staged_and_run(plan, up(x_h), up(t_h))
    del x_h
    tol = 1e-5
    orc = ftm_pairs(seed, range(B), N, K, noise, f32=True)
    near_ties = 0
    for b, o in enumerate(orc):
        for name, g in (("y1", y1), ("y2", y2), ("r1", r1), ("r2", r2)):
            ov = o[name]
            assert np.max(np.abs(g[b].astype(np.float64) - ov)) <= tol * np.max(np.abs(ov)), (name, b)
        for j, name in enumerate(("r1", "r2")):
            s = np.sort(o[name])
            if s[-1] - s[-2] > tol * np.max(np.abs(o[name])):
                assert int(res[b, j]) == o["residues"][j] == int(res_run[b, j]), (b, j)
            else:
                near_ties += 1
        for rr, kk in ((res, k), (res_run, k_run)):
            m1, m2 = int(rr[b, 0]), int(rr[b, 1])
            assert int(kk[b]) == oracle.resolve(m1, plan.M1, m2, plan.M2, N)
            if (m1, m2) == o["residues"]:
                assert int(kk[b]) == o["k"], b
    print(f"cfg3: 256 pairs within C15; {near_ties} near-tie residues; success {np.mean(k_run == k0):.3f}")


def test_cfg5_whole_signal_equals_oracle(tm):
    """cfg5 (N = 2^31, K = 65536, one pair, 5% flips): every entry of y1, y2 (the
    fold), r1, r2 (staged correlation), the residues and k (tm_run and the one-rank
    SingleSignal step) equal the oracle's Algorithm 1 on the whole signal."""
    from paper_1509_04863_b200.single import SingleSignal
    N, K, noise, seed = 2 ** 31, 65536, 0.05, 5
    plan = tm.Plan(N, K, seed=seed)
    x_h = tmgen.signal(seed, 0, N)
    t_h = tmgen.template(seed, 0, N, K, noise)
    x = torch.from_numpy(x_h).view(1, N).to(DEV)
    t = torch.from_numpy(t_h).view(1, K).to(DEV)
    y1, y2, r1, r2, res, k, res_run, k_run = staged_and_run(plan, x, t)
    ss = SingleSignal(plan, 0, 1, device=DEV)
    res_ss, k_ss = ss.step(x, t)
    torch.cuda.synchronize()
    del x
    o = oracle.ftm(x_h, t_h)
    np.testing.assert_array_equal(y1[0], o["y1"])
    np.testing.assert_array_equal(y2[0], o["y2"])
    np.testing.assert_array_equal(r1[0], o["r1"])
    np.testing.assert_array_equal(r2[0], o["r2"])
    np.testing.assert_array_equal(ss.y1.cpu().numpy()[0], o["y1"])
    np.testing.assert_array_equal(ss.y2.cpu().numpy()[0], o["y2"])
    assert tuple(res[0]) == tuple(res_run[0]) == tuple(res_ss[0].tolist()) == o["residues"]
    assert k[0] == k_run[0] == int(k_ss[0]) == o["k"]


def test_cfg5_all_ones_extreme(tm):
    """cfg5's integer extremes (reading C16): x = 1 and t = 1 give
    y_j = q = 2^15 for every entry (q1 = q2 = 32768 terms of 1; the mod-N wrap
    keeps every entry at exactly q2 terms), r_j = K q = 2^31 (beyond int32) for
    every k, residues (0, 0) (lowest-index ties, C7) and k = 0; through tm_run,
    the staged kernels and the split correlation."""
    N, K = 2 ** 31, 65536
    plan = tm.Plan(N, K, seed=0)
    q = plan.q1
    assert q == plan.q2 == 2 ** 15
    x = torch.ones((1, N), dtype=torch.int8, device=DEV)
    t = torch.ones((1, K), dtype=torch.int8, device=DEV)
    y1, y2, r1, r2, res, k, res_run, k_run = staged_and_run(plan, x, t)
    keys = plan.correlate_match_part(torch.from_numpy(y1).to(DEV), torch.from_numpy(y2).to(DEV), t, 0, 1)
    res_k, k_k = plan.match_keys(keys)
    torch.cuda.synchronize()
    assert (y1 == q).all() and (y2 == q).all()
    assert (r1 == K * q).all() and (r2 == K * q).all() and K * q == 2 ** 31
    assert tuple(res[0]) == tuple(res_run[0]) == tuple(res_k[0].tolist()) == (0, 0)
    assert k[0] == k_run[0] == int(k_k[0]) == 0


def test_general_int8_all_limbs(tm, monkeypatch):
    """General int8 data at |y| up to 127 q = 130048 (> 32767): the tensor-core
    engines split y into 4-bit limbs 0..3 plus the signed top limb (the tiled
    engine's 4-limb branch, 32767 < |y| <= 524287), and t = -128 on half the
    template; bit-exact y, r, residues and k against the oracle.
    N = 2^21, K = 2048 (q = 1024).  (The one-CTA engine takes <= 3 limbs: the
    tiled engine is forced; it is also what such a plan selects.)"""
    monkeypatch.setenv("TM_TC_TILED", "1")
    N, K, B = 2 ** 21, 2048, 3
    plan = tm.Plan(N, K, seed=9, binary=False, engine="tc")
    rng = np.random.default_rng(2048)
    x_h = rng.integers(-128, 128, (B, N)).astype(np.int8)
    x_h[0] = 127
    x_h[1, : N // 2] = -128
    t_h = rng.integers(-128, 128, (B, K)).astype(np.int8)
    t_h[0, : K // 2] = -128
    y1, y2, r1, r2, res, k, res_run, k_run = staged_and_run(plan, up(x_h), up(t_h))
    assert np.abs(y1).max() > 32767
    for b in range(B):
        o = oracle.ftm(x_h[b], t_h[b])
        for name, g in (("y1", y1), ("y2", y2), ("r1", r1), ("r2", r2)):
            np.testing.assert_array_equal(g[b], o[name], err_msg=f"{name} pair {b}")
        assert tuple(res[b]) == o["residues"] == tuple(res_run[b]) and k[b] == o["k"] == k_run[b], b


def test_fused_kernel_y_rows_every_pair(tm):
    """The fused tm_run kernel (fold + tensor-core correlation in one launch, the
    bench's cfg2 kernel): with the TM_KEEP_Y hook its folded rows y1, y2 equal the
    staged fold's (themselves pinned to the oracle above) for every pair of a full
    cfg2 batch, and its residues and k equal the staged path's."""
    N, K, B, noise, seed = 2 ** 20, 4096, 1024, 0.1, 2
    plan = tm.Plan(N, K, seed=seed, keep_y=True)
    assert plan.run_path(B) == 2
    x, t, _ = plan.generate(0, B, noise)
    ws = plan.workspace(B)
    res_run, k_run = plan.run(x, t, ws=ws)
    fy1, fy2 = plan.fold_rows(ws, B)
    y1, y2 = plan.fold(x)
    r1, r2 = plan.correlate(y1, y2, plan.fold_template(t))
    res, k = plan.match(r1, r2)
    torch.cuda.synchronize()
    assert torch.equal(fy1, y1) and torch.equal(fy2, y2)
    assert torch.equal(res_run, res) and torch.equal(k_run, k)
