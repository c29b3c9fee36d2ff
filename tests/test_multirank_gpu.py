"""One signal split over several ranks through the real CUDA path (SURVEY 8(e),
8(c.3)): every rank is a process on cuda:0 with a gloo process group (gloo
reduces CUDA tensors through host memory, so no rank's kernel ever waits on
another rank's kernel; the NCCL/NVLink path of bench.py uses the same
SingleSignal calls).  Each rank folds its chunk with tm_fold(offset, len), the
flat y1 || y2 buffer is all-reduced in place, the correlation is split by output
blocks (tm_correlate_match_part + all-reduce MAX of the keys + tm_match_keys).
Every rank must end with y1, y2, residues and k identical to the one-rank run
and to the oracle.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import tmgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
DEV = "cuda:0"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, N, K, noise, seed, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1509_04863_b200 as tm
        from paper_1509_04863_b200.single import SingleSignal
        plan = tm.Plan(N, K, seed=seed)
        ss = SingleSignal(plan, rank, world, device="cuda:0")
        x, t, k0 = plan.generate(0, 1, noise, offset=ss.offset, length=ss.length, device="cuda:0")
        for _ in range(2):   # a second step over the same buffers: no state leaks between steps
            res, k = ss.step(x, t)
        torch.cuda.synchronize()
        q.put((rank, ss.offset, ss.length, ss.y1.cpu().numpy(), ss.y2.cpu().numpy(),
               tuple(res[0].tolist()), int(k[0]), ss.split))
    except Exception as e:  # report instead of hanging the parent on q.get
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def run_ranks(world, N, K, noise, seed):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, N, K, noise, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert o[1] != "error", o
    for p in procs:
        assert p.exitcode == 0
    return sorted(out)


@pytest.fixture(scope="module")
def tm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1509_04863_b200 import _build
    _build.build()
    import paper_1509_04863_b200 as m
    return m


def one_rank(tm, N, K, noise, seed):
    from paper_1509_04863_b200.single import SingleSignal
    plan = tm.Plan(N, K, seed=seed)
    ss = SingleSignal(plan, 0, 1, device="cuda:0")
    x, t, k0 = plan.generate(0, 1, noise, device="cuda:0")
    res, k = ss.step(x, t)
    res_run, k_run = plan.run(x, t)
    torch.cuda.synchronize()
    assert tuple(res[0].tolist()) == tuple(res_run[0].tolist()) and int(k[0]) == int(k_run[0])
    return ss.y1.cpu().numpy()[0], ss.y2.cpu().numpy()[0], tuple(res[0].tolist()), int(k[0]), int(k0[0])


@pytest.mark.parametrize("world", [2, 3])
def test_split_signal_ranks_equal_oracle(tm, world):
    """N = 2^26, K = 8192 (q = 8192 rows, split into row-aligned chunks of unequal
    size at world = 3): every rank's y1, y2, residues and k equal the oracle's
    Algorithm 1 on the whole signal."""
    N, K, noise, seed = 2 ** 26, 8192, 0.05, 71
    out = run_ranks(world, N, K, noise, seed)
    x = tmgen.signal(seed, 0, N)
    t = tmgen.template(seed, 0, N, K, noise)
    o = oracle.ftm(x, t)
    pos = 0
    for rank, off, ln, y1, y2, res, k, split in out:
        assert off == pos and split
        pos += ln
        np.testing.assert_array_equal(y1[0], o["y1"], err_msg=f"rank {rank} y1")
        np.testing.assert_array_equal(y2[0], o["y2"], err_msg=f"rank {rank} y2")
        assert res == o["residues"] and k == o["k"], rank
    assert pos == N


def test_cfg5_ranks_1_2_4_8_identical(tm):
    """BASELINE cfg5 (N = 2^31, K = 65536, 5% flips): the folds, residues and k of
    2, 4 and 8 ranks are bit-identical to the one-rank run (SURVEY 8(c.3):
    "the 1-, 2-, 4- and 8-GPU runs must produce identical y (int32) and k")."""
    N, K, noise, seed = 2 ** 31, 65536, 0.05, 5
    y1, y2, res, k, k0 = one_rank(tm, N, K, noise, seed)
    torch.cuda.empty_cache()
    for world in (2, 4, 8):
        out = run_ranks(world, N, K, noise, seed)
        for rank, off, ln, a1, a2, r, kk, split in out:
            np.testing.assert_array_equal(a1[0], y1, err_msg=f"G={world} rank {rank} y1")
            np.testing.assert_array_equal(a2[0], y2, err_msg=f"G={world} rank {rank} y2")
            assert r == res and kk == k, (world, rank)


@pytest.mark.parametrize("G", [1, 2, 3])
def test_fold_reduce_emulated_ranks(tm, G):
    """tm_fold_reduce (the combine fused into the fold epilogue, SURVEY 8(f)
    f4(iii)): G ranks emulated in one process -- each chunk's fold is ADDED into
    all G destination buffers (red.global.add); afterwards every buffer holds the
    whole signal's fold, equal to tm_fold and to the oracle.  N = 2^26, K = 8192."""
    from paper_1509_04863_b200.dist import signal_chunks
    N, K, seed = 2 ** 26, 8192, 72
    plan = tm.Plan(N, K, seed=seed)
    x, t, _ = plan.generate(0, 1, 0.05)
    y1, y2 = plan.fold(x)
    bufs = [(torch.zeros((1, plan.len_y1), dtype=torch.int32, device=DEV),
             torch.zeros((1, plan.len_y2), dtype=torch.int32, device=DEV)) for _ in range(G)]
    for off, ln in signal_chunks(N, plan.M1, G):
        plan.fold_reduce(x[:, off:off + ln], [b[0] for b in bufs], [b[1] for b in bufs], offset=off, length=ln)
    torch.cuda.synchronize()
    o = oracle.ftm(tmgen.signal(seed, 0, N), tmgen.template(seed, 0, N, K, 0.05))
    for a1, a2 in bufs:
        assert torch.equal(a1, y1) and torch.equal(a2, y2)
        np.testing.assert_array_equal(a1[0].cpu().numpy(), o["y1"])
        np.testing.assert_array_equal(a2[0].cpu().numpy(), o["y2"])


def _symm_worker(port, q):
    """One-rank process group + torch symmetric memory: the fused combine through
    the real symmetric-memory buffers (the NVLS multicast address when this box
    offers one, else the peer-pointer path)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    try:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        import paper_1509_04863_b200 as tm
        from paper_1509_04863_b200.single import SingleSignal, SymmReducer
        N, K = 2 ** 26, 8192
        plan = tm.Plan(N, K, seed=73)
        x, t, _ = plan.generate(0, 1, 0.05)
        ref = SingleSignal(plan, 0, 1, device="cuda:0")
        r0, k0 = ref.step(x, t)
        out = {}
        for mc in (True, False):
            red = SymmReducer(use_multicast=mc)
            ss = SingleSignal(plan, 0, 1, device="cuda:0", reducer=red)
            multicast = red.destinations()[2]
            for _ in range(2):
                ss.fold(x)
                ss.combine()
                same = torch.equal(ss.y1, ref.y1) and torch.equal(ss.y2, ref.y2)
                r, k = ss.match(t)
                same &= torch.equal(r, r0) and torch.equal(k, k0)
                ss.flat.zero_()
            torch.cuda.synchronize()
            out["multicast" if multicast else "peer"] = bool(same)
        q.put(("ok", out))
    except Exception as e:
        q.put(("unavailable", repr(e)[:300]))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_fused_combine_symmetric_memory_one_rank(tm):
    """SingleSignal(reducer=SymmReducer()) on one rank: the fold epilogue adds into
    the symmetric-memory buffer (multicast when supported), two steps, identical to
    the plain path.  Skipped if this box offers no symmetric memory."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_symm_worker, args=(_free_port(), q))
    p.start()
    status, out = q.get(timeout=600)
    p.join(timeout=120)
    if status != "ok":
        pytest.skip(f"symmetric memory unavailable here: {out}")
    print("fused combine paths:", out)
    assert all(out.values()), out
