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


def test_ntt_constants():
    """Host-side check of the constants the NTT kernels hard-code."""
    src = open(os.path.join(ROOT, "paper_1509_04863_b200", "csrc", "correlate.cu")).read()
    p1, p2 = 2013265921, 998244353
    assert p1 == 15 * 2 ** 27 + 1 and p2 == 119 * 2 ** 23 + 1
    assert "49499719u" in src and pow(p1, -1, p2) == 49499719
    for g, p in ((31, p1), (3, p2)):
        n = p - 1
        fs = {f for f in (2, 3, 5, 7, 17) if n % f == 0}
        assert all(pow(g, n // f, p) != 1 for f in fs)
