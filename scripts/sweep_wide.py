"""Wider randomized parity sweep (not part of pytest): K up to 6000, N up to 2^22,
every engine / strategy / dtype, residues and k (and y, r) against the oracle.
usage: python scripts/sweep_wide.py first_seed last_seed"""
import os
import sys

sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
os.chdir('/root/repo')
import importlib.util  # noqa: E402

import numpy as np  # noqa: E402

spec = importlib.util.spec_from_file_location("tp", "/root/repo/tests/test_parity_gpu.py")
tp = importlib.util.module_from_spec(spec); spec.loader.exec_module(tp)
import paper_1509_04863_b200 as tm  # noqa: E402


def case(rng):
    dtype = "float32" if rng.random() < 0.2 else "int8"
    K = int(rng.integers(1, 6000))
    M = 0 if rng.random() < 0.6 else int(K + rng.integers(0, 3000))
    M1 = max(M or K, 2)
    if M == 0 and K < 2:
        M = 2
    N = int(rng.integers(max(K, 2), min(M1 * (M1 + 1) - 1, 1 << 22) + 1))
    if rng.random() < 0.5:
        N = max(M1, (N // M1) * M1)
    binary = dtype == "int8" and rng.random() < 0.7
    block = rng.random() < 0.2
    alias = (not block) and N % M1 == 0 and rng.random() < 0.2
    engine = rng.choice(["auto", "ntt"]) if dtype == "int8" else None
    return N, K, M, dtype, binary, block, alias, engine


tp._random_case = case
lo, hi = int(sys.argv[1]), int(sys.argv[2])
fails = 0
for seed in range(lo, hi):
    try:
        tp.test_randomized_sweep_against_oracle(tm, seed)
    except Exception as e:
        fails += 1
        print("FAIL seed", seed, case(np.random.default_rng(1000 + seed)), repr(e)[:300], flush=True)
        if "CUDA error" in repr(e):
            break
print("done", hi - lo, "fails", fails)
