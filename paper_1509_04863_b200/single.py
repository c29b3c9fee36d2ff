"""One huge signal split over the ranks (BASELINE cfg5).

Algorithm 1 on ONE signal x of length N whose samples are
spread over G ranks (one process per GPU) as contiguous row-aligned chunks:

1. every rank folds its chunk with global-position semantics (Eq. 2 is a sum
   over positions, so the fold of a partition is the sum of the
   folds of its parts) -- ``tm_fold(offset, len)``; the chunk holding
   position 0 also contributes the wrap and extension terms;
2. the partial y1 || y2 vectors, which live in ONE flat buffer (y1 and y2 are
   views of it), are summed IN PLACE with one all-reduce, so every rank holds
   the whole fold in the same y1 / y2 views the kernels read next;
3. the correlation is split by output blocks (8(e)(ii)): each rank runs
   ``tm_correlate_match_part`` on its part and writes one order-preserving
   key per modulus; one all-reduce MAX of the 16-byte keys and
   ``tm_match_keys`` give identical residues and k on every rank.  Plans the
   split engine does not take (fp32 data) correlate redundantly on every rank.

Fused combine (``reducer=``): instead of a fold into the
local buffer followed by an NCCL all-reduce, every rank's fold epilogue ADDS its
partial fold into all ranks' buffers at once (``tm_fold_reduce``: red.add into
peer-mapped symmetric memory, or one multimem.red into an NVLS multicast
address), so the reduction travels over NVLink while the epilogue runs and no
separate collective is launched.  Per step: barrier (every rank has zeroed its
buffer after the previous step) -> fold_reduce -> barrier (every rank's adds
have landed) -> correlation -> zero the local buffer.  ``SymmReducer`` does this
with torch symmetric memory; tests substitute a CPU stand-in.

Pipelined steps (``depth`` >= 2): consecutive steps are independent signals, so
the combine + correlation of step i runs on a side stream while the caller's
stream already folds step i+1 into the next of ``depth`` buffer sets (flat y,
workspace, keys, residues, k).  The fold kernels hold every SM, so what overlaps
is the correlation with the fold's ramp-up and tail; measured on one B200 at
cfg5: 0.357 -> 0.347 (depth 2) / 0.341 ms per step (depth 3).  ``drain`` makes
a stream wait for every outstanding step.

This module is host glue only (no arithmetic of the method); every step runs
in libtm's kernels or in the collective.  ``plan`` is a ``Plan`` (or any object
with the same methods -- the CPU wiring test stands the oracle in for it).
"""
from __future__ import annotations

from .dist import signal_chunks


def _round_up(a: int, b: int) -> int:
    return (a + b - 1) // b * b


class SingleSignal:
    """Per-rank state of the split single-signal match.

    ``rank``/``world``/``group``: the process group the chunks are spread over
    (world = 1: no collective).  ``split_correlation``: None = split when the
    plan is int8 and world > 1.  Buffers are allocated once on ``device``.
    """

    def __init__(self, plan, rank: int = 0, world: int = 1, group=None, device="cuda",
                 split_correlation: bool | None = None, reducer=None, depth: int = 1):
        import torch
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        self.offset, self.length = signal_chunks(plan.N, plan.M1, world)[rank]
        n1, n2 = int(plan.len_y1), int(plan.len_y2)
        # y1 region padded to 32 entries (128 B) so y2 starts 16-byte aligned for the
        # kernels' vector loads; the padding is zero and never read.
        self.ldy1 = _round_up(n1, 32)
        self.reducer = reducer
        if depth < 1 or (depth > 1 and reducer is not None):
            raise ValueError("depth >= 1; the fused combine (reducer=) runs unpipelined (depth 1)")
        self.depth = int(depth)
        self._slots = []
        for _ in range(self.depth):
            if reducer is None:
                flat = torch.zeros(self.ldy1 + n2, dtype=plan.y_dtype, device=device)
            else:   # symmetric (peer-visible) buffer, zeroed, owned by the reducer
                flat = reducer.make_flat(self.ldy1 + n2, plan.y_dtype, device, self.ldy1)
            self._slots.append({
                "flat": flat, "y1": flat[:n1].view(1, n1), "y2": flat[self.ldy1:].view(1, n2),
                "ws": plan.workspace(1, device),
                "keys": torch.empty((1, 2), dtype=torch.int64, device=device),
                "residues": torch.empty((1, 2), dtype=torch.int32, device=device),
                "k": torch.empty(1, dtype=torch.int64, device=device)})
        self._use(0)
        self._i = 0
        self._side = self._folded = self._done = None
        if self.depth > 1 and torch.device(device).type == "cuda":
            self._side = torch.cuda.Stream(device=device)
            self._folded = [torch.cuda.Event() for _ in range(self.depth)]
            self._done = [torch.cuda.Event() for _ in range(self.depth)]
            for e in self._done:
                e.record(self._side)
        if split_correlation is None:
            split_correlation = world > 1 and getattr(plan, "dtype", 0) == 0  # TM_I8
        self.split = bool(split_correlation) and world > 1

    def _use(self, b: int):
        """Make buffer set b the current one (flat / y1 / y2 / ws / keys / residues / k)."""
        for name, v in self._slots[b].items():
            setattr(self, name, v)

    @property
    def reduce_bytes(self) -> int:
        return self.flat.numel() * self.flat.element_size()

    def fold(self, x_chunk, stream=None):
        """Step 3 on this rank's chunk: the partial fold into the y1 / y2 views, or
        (fused combine) added into every rank's buffer by the fold's epilogue."""
        if self.reducer is not None:
            self.reducer.barrier()   # every rank has zeroed its buffer since it last read it
            d1, d2, mc = self.reducer.destinations()
            self.plan.fold_reduce(x_chunk, d1, d2, offset=self.offset, length=self.length, multicast=mc,
                                  ws=self.ws, stream=stream)
            return
        self.plan.fold(x_chunk, offset=self.offset, length=self.length, y1=self.y1, y2=self.y2,
                       accumulate=False, ws=self.ws, stream=stream)

    def combine(self):
        """Sum the partial folds over the ranks in place (one all-reduce of y1 || y2);
        fused combine: wait until every rank's adds have landed."""
        if self.reducer is not None:
            self.reducer.barrier()
            return
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)

    def match(self, t, stream=None):
        """Steps 4-9 on the combined fold: residues [1][2] int32, k [1] int64 on every rank."""
        if self.split:
            import torch.distributed as dist
            self.plan.correlate_match_part(self.y1, self.y2, t, self.rank, self.world, keys=self.keys,
                                           ws=self.ws, stream=stream)
            dist.all_reduce(self.keys, op=dist.ReduceOp.MAX, group=self.group)
            self.plan.match_keys(self.keys, residues=self.residues, k=self.k, stream=stream)
        else:
            self.plan.correlate_match(self.y1, self.y2, t, residues=self.residues, k=self.k, ws=self.ws,
                                      stream=stream)
        return self.residues, self.k

    def step(self, x_chunk, t, stream=None, events=None):
        """One whole pass: fold -> all-reduce -> correlate / argmax / CRT.
        ``events``: optional 4 CUDA events recorded between the stages.
        depth >= 2: returns this step's (residues, k) buffers, complete once the side
        stream has finished them -- ``drain(stream)`` before reading."""
        import contextlib

        import torch
        if self.depth > 1:
            return self._step_pipelined(x_chunk, t, stream, events)
        ctx = torch.cuda.stream(stream) if stream is not None and hasattr(stream, "cuda_stream") \
            else contextlib.nullcontext()
        with ctx:
            if events:
                events[0].record()
            self.fold(x_chunk, stream=stream)
            if events:
                events[1].record()
            self.combine()
            if events:
                events[2].record()
            out = self.match(t, stream=stream)
            if events:
                events[3].record()
            if self.reducer is not None:
                self.flat.zero_()   # ready for the next step's adds (ordered by its first barrier)
        return out

    def _step_pipelined(self, x_chunk, t, stream, events):
        import torch
        b = self._i % self.depth
        self._i += 1
        self._use(b)
        if self._side is None:   # CPU stand-in (wiring tests): the buffer sets rotate, nothing overlaps
            self.fold(x_chunk)
            self.combine()
            return self.match(t)
        cs = stream if stream is not None and hasattr(stream, "cuda_stream") else torch.cuda.current_stream()
        cs.wait_event(self._done[b])   # buffer set b is free once step i - depth has finished with it
        if events:
            events[0].record(cs)
        self.fold(x_chunk, stream=cs)
        if events:
            events[1].record(cs)
        self._folded[b].record(cs)
        self._side.wait_event(self._folded[b])
        with torch.cuda.stream(self._side):   # the collectives order themselves on the current stream
            self.combine()
            if events:
                events[2].record(self._side)
            out = self.match(t, stream=self._side)
            if events:
                events[3].record(self._side)
        self._done[b].record(self._side)
        return out

    def drain(self, stream=None):
        """Make ``stream`` (default: the current one) wait for every outstanding
        pipelined step; afterwards ``residues`` / ``k`` hold the latest step's result."""
        if self._side is None:
            return
        import torch
        cs = stream if stream is not None and hasattr(stream, "cuda_stream") else torch.cuda.current_stream()
        for e in self._done:
            cs.wait_event(e)


class SymmReducer:
    """Fused combine over torch symmetric memory (NVLink peer mappings; NVLS
    multicast when the system supports it).  One per process group."""

    def __init__(self, group=None, use_multicast: bool = True):
        import torch.distributed as dist
        self.group = group if group is not None else dist.group.WORLD
        self.use_multicast = use_multicast
        self.handle = None

    def make_flat(self, n, dtype, device, ldy1):
        import torch.distributed._symmetric_memory as symm
        flat = symm.empty(n, dtype=dtype, device=device)
        flat.zero_()
        self.handle = symm.rendezvous(flat, self.group.group_name)
        self.ldy1, self.esize = ldy1, flat.element_size()
        self.handle.barrier(channel=0)
        return flat

    def destinations(self):
        h, off2 = self.handle, self.ldy1 * self.esize
        if self.use_multicast and h.has_multicast_support and h.multicast_ptr:
            return [h.multicast_ptr], [h.multicast_ptr + off2], True
        return list(h.buffer_ptrs), [p + off2 for p in h.buffer_ptrs], False

    def barrier(self):
        self.handle.barrier(channel=0)
