"""CPU checks of the C-ABI library: it loads, exports every symbol include/tm.h
declares, and its host-side constants are right.  No compute calls (no GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "tm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(tm_[a-z_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def libtm():
    from paper_1509_04863_b200 import _build
    _build.build()
    import paper_1509_04863_b200 as tm
    return tm


def test_header_declares_expected_calls():
    names = declared_symbols()
    for want in ("tm_plan_create", "tm_fold", "tm_fold_template", "tm_correlate", "tm_match", "tm_run"):
        assert want in names


def test_library_exports_every_declared_symbol(libtm):
    out = subprocess.check_output(["nm", "-D", "--defined-only", libtm.lib_path()]).decode()
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(libtm.EXPORTED_SYMBOLS) == set(declared_symbols())
    L = libtm.lib()
    for s in declared_symbols():
        getattr(L, s)


def test_library_is_sm100a(libtm):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libtm.lib_path()]).decode()
    assert "sm_100a" in out


def test_status_strings(libtm):
    L = libtm.lib()
    assert L.tm_status_string(0) == b"TM_OK"
    assert L.tm_status_string(1) == b"TM_EINVAL"


def test_plan_create_rejects_invalid_without_gpu(libtm):
    """Argument checks are synchronous and precede any CUDA call."""
    import ctypes
    L = libtm.lib()
    h = ctypes.c_void_p()
    assert L.tm_plan_create(ctypes.byref(h), 1024, 16, 0, 0, 0, 1) == 1   # 16*17 <= 1024
    assert b"smallest valid M1 is 32" in L.tm_last_error()
    assert L.tm_plan_create(ctypes.byref(h), 1024, 40, 32, 0, 0, 1) == 1  # M1 < K
    assert L.tm_plan_create(ctypes.byref(h), 0, 4, 0, 0, 0, 0) == 1
    assert L.tm_plan_create(ctypes.byref(h), 1024, 64, 0, 0, 1, 1) == 1   # TM_BINARY needs int8
    assert L.tm_plan_create(ctypes.byref(h), 1024, 64, 0, 0, 0, 16 | 8) == 1  # TM_BLOCK excludes TM_ALIAS_REPAIR
    assert L.tm_plan_create(ctypes.byref(h), 1024, 64, 0, 0, 0, 128) == 1  # unknown flag
    assert L.tm_plan_create(ctypes.byref(h), 1001, 40, 0, 0, 0, 8) == 2    # TM_ALIAS_REPAIR needs M1 | N
    M = (ctypes.c_int64 * 3)(17, 18, 20)                                      # 18, 20 not co-prime
    L.tm_mplan_create.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int,
                                  ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32]
    assert L.tm_mplan_create(ctypes.byref(h), 4096, 16, M, 3, 0, 0, 1) == 1
    assert b"co-prime" in L.tm_last_error()
    M = (ctypes.c_int64 * 2)(17, 18)                                          # 306 <= N
    assert L.tm_mplan_create(ctypes.byref(h), 4096, 16, M, 2, 0, 0, 1) == 1
    M = (ctypes.c_int64 * 3)(15, 17, 19)                                      # 15 < K
    assert L.tm_mplan_create(ctypes.byref(h), 4096, 16, M, 3, 0, 0, 1) == 1
    assert L.tm_mplan_create(ctypes.byref(h), 4096, 16, M, 1, 0, 0, 1) == 1   # alpha < 2


def test_ntt_constants():
    """Host-side check of the constants the NTT kernels hard-code (tm_internal.cuh)."""
    src = open(os.path.join(ROOT, "paper_1509_04863_b200", "csrc", "tm_internal.cuh")).read()
    consts = dict(re.findall(r"#define (TM_P\w+) (\d+)u", src))
    p1, p2 = int(consts["TM_P1"]), int(consts["TM_P2"])
    assert p1 == 479 * 2 ** 21 + 1 and p2 == 119 * 2 ** 23 + 1
    assert p1 < 2 ** 30 and p2 < 2 ** 30          # lazy reduction needs 4p < 2^32
    assert int(consts["TM_P1_PINV"]) == (-pow(p1, -1, 2 ** 32)) % 2 ** 32
    assert int(consts["TM_P2_PINV"]) == (-pow(p2, -1, 2 ** 32)) % 2 ** 32
    assert int(re.search(r"TM_P1_INV_MOD_P2 (\d+)ull", src).group(1)) == pow(p1, -1, p2)
    for p, fs in ((p1, (2, 479)), (p2, (2, 7, 17))):
        assert all((p - 1) % f == 0 for f in fs)
        n = p - 1
        m = n
        for f in fs:
            while m % f == 0:
                m //= f
        assert m == 1                                # complete factorisation of p - 1
        assert all(pow(3, n // f, p) != 1 for f in fs)  # 3 is a primitive root
