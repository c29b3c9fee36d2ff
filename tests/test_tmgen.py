"""Host input generator (tmgen/): determinism and the workload's statistics."""
import numpy as np

import tmgen


def test_signal_values_and_determinism():
    a = tmgen.signal(7, 3, 4096)
    b = tmgen.signal(7, 3, 4096)
    np.testing.assert_array_equal(a, b)
    assert set(np.unique(a)) <= {-1, 1}
    assert not np.array_equal(a, tmgen.signal(7, 4, 4096))
    assert not np.array_equal(a, tmgen.signal(8, 3, 4096))
    # sub-range generation is the same stream
    np.testing.assert_array_equal(tmgen.signal(7, 3, 4096, lo=100, length=333), a[100:433])


def test_signal_balanced():
    n = 10 ** 6
    x = tmgen.signal(1, 0, n).astype(np.int64)
    assert abs(x.mean()) < 5 / np.sqrt(n)


def test_template_is_planted_window():
    N, K = 5000, 300
    for pair in range(4):
        x = tmgen.signal(5, pair, N)
        k0 = tmgen.k0(5, pair, N)
        assert 0 <= k0 < N
        t = tmgen.template(5, pair, N, K, 0.0)
        np.testing.assert_array_equal(t, x[(k0 + np.arange(K)) % N])
        t1 = tmgen.template(5, pair, N, K, 1.0)
        np.testing.assert_array_equal(t1, -t)


def test_flip_rate():
    N, K = 2 ** 16, 2 ** 15
    x = tmgen.signal(9, 0, N)
    k0 = tmgen.k0(9, 0, N)
    t = tmgen.template(9, 0, N, K, 0.1)
    flips = np.mean(t != x[(k0 + np.arange(K)) % N])
    assert abs(flips - 0.1) < 5 * np.sqrt(0.09 / K)


def test_k0_uniform():
    N = 1000
    ks = np.array([tmgen.k0(3, b, N) for b in range(20000)])
    hist = np.bincount(ks // 100, minlength=10)
    assert hist.min() > 1700 and hist.max() < 2300


def test_gaussian_signal():
    x = tmgen.signal(2, 0, 200000, dtype=np.float32)
    assert x.dtype == np.float32
    assert abs(x.mean()) < 0.02 and abs(x.var() - 1) < 0.02
    N, K = 4096, 512
    t = tmgen.template(2, 1, N, K, 0.5, dtype=np.float32)
    xs = tmgen.signal(2, 1, N, dtype=np.float32)
    k0 = tmgen.k0(2, 1, N)
    d = t.astype(np.float64) - xs[(k0 + np.arange(K)) % N]
    assert abs(d.std() - 0.5) < 0.06


def test_batch_matches_single():
    x, t, k = tmgen.batch(4, 10, 3, 1024, 64, 0.2)
    for b in range(3):
        np.testing.assert_array_equal(x[b], tmgen.signal(4, 10 + b, 1024))
        np.testing.assert_array_equal(t[b], tmgen.template(4, 10 + b, 1024, 64, 0.2))
        assert k[b] == tmgen.k0(4, 10 + b, 1024)
