"""Multi-rank host logic on CPU (gloo, world_size 2): the partition of one signal
into row-aligned chunks, the all-reduce of partial folds (partial folds computed
by the oracle stand in for tm_fold on each rank), batch sharding by global pair
index, and the max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1509_04863_b200 import dist as tmdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_signal_chunks_partition():
    for N, M1, G in ((2 ** 31, 65536, 8), (4096 * 37, 4096, 3), (4096, 256, 5), (1024, 256, 4)):
        ch = tmdist.signal_chunks(N, M1, G)
        assert len(ch) == G
        pos = 0
        for off, ln in ch:
            assert off == pos and off % M1 == 0 and ln % M1 == 0
            pos += ln
        assert pos == N
        lens = [ln for _, ln in ch]
        assert max(lens) - min(lens) <= M1
    with pytest.raises(ValueError):
        tmdist.signal_chunks(1000, 64, 2)


def test_pair_range():
    assert tmdist.pair_range(1024, 0) == (0, 1024)
    assert tmdist.pair_range(1024, 3) == (3072, 1024)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import tmgen
        N, K = 64 * 48, 64           # M1 = 64, M2 = 65, q = 48
        M1, M2 = oracle.moduli(N, K)
        x = tmgen.signal(9, 0, N)
        off, ln = tmdist.signal_chunks(N, M1, world)[rank]
        y1 = torch.from_numpy(oracle.fold(x, M1, K, off, ln))
        y2 = torch.from_numpy(oracle.fold(x, M2, K, off, ln))
        ret = tmdist.allreduce_folds(y1, y2)
        assert ret[0] is y1 and ret[1] is y2          # in place: the caller's tensors hold the sum
        ok_fold = np.array_equal(y1.numpy(), oracle.fold(x, M1, K)) and np.array_equal(y2.numpy(), oracle.fold(x, M2, K))
        # every rank then matches the same full fold -> identical k on all ranks
        t = tmgen.template(9, 0, N, K, 0.0)
        r1 = oracle.correlate(y1.numpy(), M1, t)
        r2 = oracle.correlate(y2.numpy(), M2, t)
        z = oracle.crt(oracle.argmax(r1), M1, oracle.argmax(r2), M2)
        k = z if z < N else -1
        ks = [None] * world
        dist.all_gather_object(ks, k)
        tmax = tmdist.max_over_ranks(1.0 + rank)
        # split correlation (8(e)(ii)): each rank's best (r, k) over its half of the
        # outputs as the documented int64 key, one all-reduce MAX, decode
        def key(r, kk):
            v = (((int(r) + (1 << 42)) << 21) | ((1 << 21) - 1 - int(kk))) ^ (1 << 63)
            return v - (1 << 64) if v >= (1 << 63) else v
        keys = []
        for r in (r1, r2):
            lo, hi = len(r) * rank // world, len(r) * (rank + 1) // world
            kk = lo + int(np.argmax(r[lo:hi]))
            keys.append(key(r[kk], kk))
        keys = torch.tensor([keys], dtype=torch.int64)
        tmdist.allreduce_max_keys(keys)
        dec = [((1 << 21) - 1 - ((int(v) + (1 << 64)) % (1 << 64) & ((1 << 21) - 1))) for v in keys[0]]
        ok_keys = dec == [oracle.argmax(r1), oracle.argmax(r2)]
        q.put((rank, ok_fold and ok_keys, ks, k == oracle.ftm(x, t)["k"], tmax))
    finally:
        dist.destroy_process_group()


def test_allreduce_of_partial_folds_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_fold, ks, ok_k, tmax in res:
        assert ok_fold, rank
        assert len(set(ks)) == 1
        assert ok_k
        assert tmax == 2.0


# --------------------------------------------------------------------------------
# SingleSignal (paper_1509_04863_b200/single.py) wiring on gloo ranks, with the
# oracle standing in for libtm's kernels (this is a test of the host logic: the
# in-place all-reduce of the flat y1 || y2 buffer, the split correlation keys).
class OraclePlan:
    """Duck-typed Plan whose entry points run the oracle on CPU tensors."""

    def __init__(self, N, K):
        import oracle
        self.N, self.K = N, K
        self.M1, self.M2 = oracle.moduli(N, K)
        self.len_y1, self.len_y2 = self.M1 + K, self.M2 + K
        self.y_dtype, self.dtype = torch.int32, 0
        self.calls = []

    def workspace(self, batch, device):
        return torch.empty(1, dtype=torch.uint8)

    def fold(self, x, offset, length, y1, y2, accumulate, ws, stream):
        import oracle
        assert not accumulate
        xfull = np.zeros(self.N, np.int8)          # global positions; outside the chunk unused
        xfull[offset:offset + length] = x[0].numpy()
        y1.copy_(torch.from_numpy(oracle.fold(xfull, self.M1, self.K, offset, length)).view(1, -1))
        y2.copy_(torch.from_numpy(oracle.fold(xfull, self.M2, self.K, offset, length)).view(1, -1))
        self.calls.append("fold")

    @staticmethod
    def _key(r, k):
        v = (((int(r) + (1 << 42)) << 21) | ((1 << 21) - 1 - int(k))) ^ (1 << 63)
        return v - (1 << 64) if v >= (1 << 63) else v

    def correlate_match_part(self, y1, y2, t, part, nparts, keys, ws, stream):
        import oracle
        out = []
        for y, M in ((y1, self.M1), (y2, self.M2)):
            r = oracle.correlate(y[0].numpy().astype(np.int64), M, t[0].numpy())
            lo, hi = M * part // nparts, M * (part + 1) // nparts
            kk = lo + int(np.argmax(r[lo:hi]))
            out.append(self._key(r[kk], kk))
        keys.copy_(torch.tensor([out], dtype=torch.int64))
        self.calls.append("part")

    def match_keys(self, keys, residues, k, stream):
        import oracle
        dec = [(1 << 21) - 1 - ((int(v) + (1 << 64)) % (1 << 64) & ((1 << 21) - 1)) for v in keys[0]]
        residues.copy_(torch.tensor([dec], dtype=torch.int32))
        z = oracle.crt(dec[0], self.M1, dec[1], self.M2)
        k.fill_(z if z < self.N else -1)
        self.calls.append("keys")

    def correlate_match(self, y1, y2, t, residues, k, ws, stream):
        import oracle
        r1 = oracle.correlate(y1[0].numpy().astype(np.int64), self.M1, t[0].numpy())
        r2 = oracle.correlate(y2[0].numpy().astype(np.int64), self.M2, t[0].numpy())
        m1, m2 = oracle.argmax(r1), oracle.argmax(r2)
        residues.copy_(torch.tensor([[m1, m2]], dtype=torch.int32))
        z = oracle.crt(m1, self.M1, m2, self.M2)
        k.fill_(z if z < self.N else -1)
        self.calls.append("whole")


def _single_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import tmgen
        from paper_1509_04863_b200.single import SingleSignal
        N, K = 64 * 45, 64
        plan = OraclePlan(N, K)
        ss = SingleSignal(plan, rank, world, device="cpu")
        x = tmgen.signal(13, 0, N)
        t = tmgen.template(13, 0, N, K, 0.05)
        xc = torch.from_numpy(x[ss.offset:ss.offset + ss.length].copy()).view(1, -1)
        res, k = ss.step(xc, torch.from_numpy(t).view(1, -1))
        o = oracle.ftm(x, t)
        ok = (np.array_equal(ss.y1[0].numpy(), o["y1"]) and np.array_equal(ss.y2[0].numpy(), o["y2"])
              and tuple(res[0].tolist()) == o["residues"] and int(k[0]) == o["k"])
        q.put((rank, ok, plan.calls, ss.offset, ss.length))
    finally:
        dist.destroy_process_group()


def _single_depth_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import tmgen
        from paper_1509_04863_b200.single import SingleSignal
        N, K = 64 * 30, 64
        ss = SingleSignal(OraclePlan(N, K), rank, world, device="cpu", depth=2)
        ok, held = True, []
        for i in range(3):          # three different signals through two rotating buffer sets
            x = tmgen.signal(21 + i, 0, N)
            t = tmgen.template(21 + i, 0, N, K, 0.05)
            xc = torch.from_numpy(x[ss.offset:ss.offset + ss.length].copy()).view(1, -1)
            res, k = ss.step(xc, torch.from_numpy(t).view(1, -1))
            o = oracle.ftm(x, t)
            ok = ok and (np.array_equal(ss.y1[0].numpy(), o["y1"]) and np.array_equal(ss.y2[0].numpy(), o["y2"])
                         and tuple(res[0].tolist()) == o["residues"] and int(k[0]) == o["k"])
            held.append((k, o["k"]))
        # step 1's result (slot 1) is still intact after step 2 wrote slot 0
        ok = ok and int(held[1][0][0]) == held[1][1] and held[0][0] is held[2][0]
        ss.drain()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_single_signal_depth_rotates_buffers_gloo():
    """SingleSignal(depth=2) on two gloo ranks: the buffer sets rotate, every step's
    all-reduce and keys use the current set, and a result stays valid until its
    set comes round again."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_single_depth_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res


@pytest.mark.parametrize("world", [2, 3])
def test_single_signal_wiring_gloo(world):
    """Each rank folds its chunk, the flat y1 || y2 buffer is all-reduced in place,
    the split correlation's keys are MAX-reduced: every rank's y1, y2, residues
    and k equal the oracle's whole-signal Algorithm 1."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_single_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    covered = 0
    for rank, ok, calls, off, ln in sorted(res):
        assert ok, rank
        assert calls == ["fold", "part", "keys"], calls
        assert off == covered
        covered += ln
    assert covered == 64 * 45


# --------------------------------------------------------------------------------
# Fused combine (SingleSignal(reducer=...), tm_fold_reduce):
# the protocol -- barrier, every rank ADDS its partial fold into every rank's
# buffer, barrier, correlate, zero -- on gloo ranks with CPU shared-memory buffers
# standing in for symmetric memory and the oracle standing in for the kernels.
class SharedCpuReducer:
    def __init__(self, bufs, rank, lock):
        self.bufs, self.rank, self.lock = bufs, rank, lock

    def make_flat(self, n, dtype, device, ldy1):
        assert self.bufs[self.rank].numel() == n
        self.ldy1 = ldy1
        return self.bufs[self.rank]

    def destinations(self):
        return ([b[:self.n1] for b in self.bufs], [b[self.ldy1:] for b in self.bufs], False)

    def barrier(self):
        dist.barrier()


class OracleReducePlan(OraclePlan):
    def __init__(self, N, K, lock):
        super().__init__(N, K)
        self.lock = lock

    def fold_reduce(self, x, d1, d2, offset, length, multicast, ws, stream):
        import oracle
        xfull = np.zeros(self.N, np.int8)
        xfull[offset:offset + length] = x[0].numpy()
        p1 = torch.from_numpy(oracle.fold(xfull, self.M1, self.K, offset, length)).to(torch.int32)
        p2 = torch.from_numpy(oracle.fold(xfull, self.M2, self.K, offset, length)).to(torch.int32)
        with self.lock:  # the device's red.add is atomic; CPU stand-in: one writer at a time
            for a, b in zip(d1, d2):
                a.add_(p1)
                b.add_(p2)
        self.calls.append("fold_reduce")


def _fused_worker(rank, world, port, bufs, lock, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import tmgen
        from paper_1509_04863_b200.single import SingleSignal
        N, K = 64 * 45, 64
        plan = OracleReducePlan(N, K, lock)
        red = SharedCpuReducer(bufs, rank, lock)
        red.n1 = plan.len_y1
        ss = SingleSignal(plan, rank, world, device="cpu", reducer=red)
        ok = True
        for seed in (13, 14):   # two steps: the buffers must be re-zeroed between them
            x = tmgen.signal(seed, 0, N)
            t = tmgen.template(seed, 0, N, K, 0.05)
            xc = torch.from_numpy(x[ss.offset:ss.offset + ss.length].copy()).view(1, -1)
            ss.fold(xc)
            ss.combine()
            y1, y2 = ss.y1[0].clone().numpy(), ss.y2[0].clone().numpy()
            res, k = ss.match(torch.from_numpy(t).view(1, -1))
            ss.flat.zero_()
            o = oracle.ftm(x, t)
            ok &= (np.array_equal(y1, o["y1"]) and np.array_equal(y2, o["y2"]) and
                   tuple(res[0].tolist()) == o["residues"] and int(k[0]) == o["k"])
        q.put((rank, ok, plan.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_single_signal_fused_combine_gloo(world):
    """Every rank adds its partial fold into every rank's buffer (the fused
    combine's protocol); after the second barrier each buffer holds the whole
    fold, and residues and k equal the oracle's, on two consecutive steps."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    lock = ctx.Lock()
    N, K = 64 * 45, 64
    n = (64 + K + 31) // 32 * 32 + 65 + K
    bufs = [torch.zeros(n, dtype=torch.int32).share_memory_() for _ in range(world)]
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, bufs, lock, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, calls in res:
        assert ok, rank
        assert calls.count("fold_reduce") == 2 and "part" in calls
