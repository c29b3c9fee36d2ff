"""Templates longer than 2^17 (Fig. 1a runs K up to 2^25 at N = 2^26,
P:328; SURVEY 8(d)'s cfg5 companions K = 2^18, 2^19 and cfg4's K = 32768, 65536).
The NTT engine's tables stop at transforms of 2^18, so these plans correlate on
the tiled tensor-core engine; parity against the oracle: whole vectors where the
oracle's K*M direct correlation finishes in about a minute, sampled outputs
(or_correlate_at, the same formula one output at a time, pinned in
test_oracle.py) at N = 2^31.
"""
import numpy as np
import pytest

import oracle
import tmgen

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


def gpu_all(plan, x, t):
    y1, y2 = plan.fold(x)
    r1, r2 = plan.correlate(y1, y2, plan.fold_template(t))
    res, k = plan.match(r1, r2)
    res_run, k_run = plan.run(x, t)
    torch.cuda.synchronize()
    return [v.cpu().numpy() for v in (y1, y2, r1, r2, res, k, res_run, k_run)]


def test_plan_beyond_ntt_tables(tm):
    """K = 2^18 binary int8: the plan is accepted and correlates on the tensor
    cores; general int8 data at that K (|r| per limb beyond int32) and fp32 have
    their own engines or are rejected with TM_EUNSUPPORTED, never a wrong result."""
    p = tm.Plan(2 ** 31, 2 ** 18)
    assert p.corr_engine == 1 and p.L2 == 2 ** 19   # > 2^18: beyond the NTT tables
    with pytest.raises(tm.TMError):
        tm.Plan(2 ** 25, 2 ** 18, binary=False)
    with pytest.raises(tm.TMError):
        tm.Plan(2 ** 25, 2 ** 18, engine="ntt")


def test_k_2e18_whole_vectors(tm):
    """N = 2^25, K = 2^18 (q = 128), +-1 data, 5% flips, two pairs: y1, y2, r1, r2,
    residues and k byte-identical to the oracle (its direct correlation is 2 K M =
    2^37 MAC, about a minute)."""
    N, K, seed = 2 ** 25, 2 ** 18, 181
    plan = tm.Plan(N, K, seed=seed)
    x_h, t_h, k0 = tmgen.batch(seed, 0, 2, N, K, 0.05)
    y1, y2, r1, r2, res, k, res_run, k_run = gpu_all(plan, torch.from_numpy(x_h).to(DEV),
                                                     torch.from_numpy(t_h).to(DEV))
    from oracle_pool import ftm_pairs
    for b, o in enumerate(ftm_pairs(seed, range(2), N, K, 0.05)):
        for n, g in (("y1", y1), ("y2", y2), ("r1", r1), ("r2", r2)):
            np.testing.assert_array_equal(g[b], o[n], err_msg=f"{n} pair {b}")
        assert tuple(res[b]) == o["residues"] == tuple(res_run[b]) and k[b] == o["k"] == k_run[b]
    assert (k_run == k0).all()  # q = 128: far inside the success regime (K^2 / log K >> N)


@pytest.mark.parametrize("K", [2 ** 18, 2 ** 19])
def test_cfg5_companions_sampled(tm, K):
    """cfg5 signal (N = 2^31, 5% flips) with K = 2^18 and 2^19: every entry of
    y1, y2 against the oracle's Eq. 2 fold; r1, r2 on 300 sampled outputs (incl.
    the GPU's argmax positions and the planted shift's bins) against
    or_correlate_at on the oracle's fold; the residues are the lowest-index
    argmax of the GPU's r (checked whole on the host) and k = CRT(residues)."""
    N, seed = 2 ** 31, 5
    plan = tm.Plan(N, K, seed=seed)
    x_h = tmgen.signal(seed, 0, N)
    t_h = tmgen.template(seed, 0, N, K, 0.05)
    k0 = tmgen.k0(seed, 0, N)
    y1, y2, r1, r2, res, k, res_run, k_run = gpu_all(plan, torch.from_numpy(x_h).view(1, N).to(DEV),
                                                     torch.from_numpy(t_h).view(1, K).to(DEV))
    rng = np.random.default_rng(K)
    for j, (M, y, r) in enumerate(((plan.M1, y1, r1), (plan.M2, y2, r2))):
        oy = oracle.fold(x_h, M, K)
        np.testing.assert_array_equal(y[0], oy, err_msg=f"y{j + 1}")
        ks = np.unique(np.concatenate([rng.integers(0, M, 296), [0, M - 1, int(res[0, j]), k0 % M]]))
        np.testing.assert_array_equal(r[0][ks], oracle.correlate_at(oy, t_h, ks), err_msg=f"r{j + 1}")
        m = int(np.flatnonzero(r[0] == r[0].max())[0])
        assert m == int(res[0, j]) == int(res_run[0, j])
    z = oracle.crt(int(res[0, 0]), plan.M1, int(res[0, 1]), plan.M2)
    assert k[0] == k_run[0] == (z if z < N else -1)
    print(f"K = {K}: k = {int(k_run[0])}, planted {k0}")


@pytest.mark.parametrize("N,K", [(2 ** 20, 16384), (2 ** 22, 32768), (2 ** 26, 65536), (2 ** 24, 131072)])
def test_f32_four_step_fft(tm, N, K):
    """fp32 correlations whose transform exceeds one CTA's registers (L2 = 2^15 ..
    2^18; (2^26, 2^16) is PAPER.md Table 2's shape): the four-step FFT
    (pass A across 2^14-entry segments, pass B per segment) under reading C15
    against the oracle's fp64 direct correlation, one pair each."""
    from test_parity_gpu import check_f32_pairs
    plan = tm.Plan(N, K, seed=151, dtype="float32")
    assert plan.L2 > 2 ** 14
    x_h, t_h, _ = tmgen.batch(151, 0, 1, N, K, 0.5, dtype=np.float32)
    check_f32_pairs(tm, plan, x_h, t_h, [0])
