"""Consecutive batches software-pipelined over two streams (host glue only).

Algorithm 1's steps of ONE batch depend on each other (fold -> correlation ->
argmax -> CRT), but consecutive batches do not.  The staged
paths run the fold as a persistent HBM-bound kernel and the correlation on the
tensor cores (or the FFT / NTT engines) afterwards, each leaving the other's
resource idle.  ``Pipeline.step`` enqueues the fold of batch i on the caller's
stream and the correlation + match of batch i on a side stream, with ``depth``
sets of intermediate buffers (y1, y2, workspace) and results, so the fold of batch
i+1 starts while batch i is still being correlated.  Measured on one B200
(`scripts/pipeline_probe.py`, per step): cfg4 K = 16384 0.238 -> 0.226 ms,
K = 32768 0.315 -> 0.295, cfg3 0.734 -> 0.720; the fused one-kernel path (cfg2)
already overlaps the two inside the kernel and is run as is.

No arithmetic of the method lives here: every step runs in libtm's kernels.
"""
from __future__ import annotations


class Pipeline:
    """``depth`` batches of ``batch`` pairs in flight on ``plan``'s device.

    step(x, t) -> (residues, k): buffers of this step's slot, complete once the
    side stream has finished them -- call ``drain(stream)`` (or wait on
    ``done_event(slot)``) before reading; they are reused ``depth`` steps later.
    """

    def __init__(self, plan, batch: int, depth: int = 2, device="cuda"):
        import torch
        if depth < 1:
            raise ValueError("depth >= 1")
        self.plan, self.batch, self.depth = plan, int(batch), int(depth)
        self.fused = plan.run_path(batch) in (2, 3)   # one kernel per step (fused / small pair): nothing to split
        dev = torch.device(device)
        self._slots = []
        for _ in range(self.depth):
            slot = {"ws": plan.workspace(batch, dev),
                    "residues": torch.empty((batch, 2), dtype=torch.int32, device=dev),
                    "k": torch.empty(batch, dtype=torch.int64, device=dev)}
            if not self.fused:
                slot["y1"] = torch.empty((batch, plan.len_y1), dtype=plan.y_dtype, device=dev)
                slot["y2"] = torch.empty((batch, plan.len_y2), dtype=plan.y_dtype, device=dev)
            self._slots.append(slot)
        self._side = torch.cuda.Stream(device=dev)
        self._folded = [torch.cuda.Event() for _ in range(self.depth)]
        self._done = [torch.cuda.Event() for _ in range(self.depth)]
        for e in self._done:
            e.record(self._side)
        self._i = 0
        self.last_slot = 0

    def step(self, x, t, stream=None):
        import torch
        if x.shape[0] != self.batch:
            raise ValueError("Pipeline.step: batch differs from the one the buffers were sized for")
        cs = stream if stream is not None and hasattr(stream, "cuda_stream") else torch.cuda.current_stream()
        b = self._i % self.depth
        self._i += 1
        self.last_slot = b
        s = self._slots[b]
        if self.fused or self.depth == 1:
            return self.plan.run(x, t, residues=s["residues"], k=s["k"], ws=s["ws"], stream=cs)
        cs.wait_event(self._done[b])   # slot b is free once step i - depth has finished with it
        self.plan.fold(x, y1=s["y1"], y2=s["y2"], ws=s["ws"], stream=cs)
        self._folded[b].record(cs)
        self._side.wait_event(self._folded[b])
        self.plan.correlate_match(s["y1"], s["y2"], t, residues=s["residues"], k=s["k"], ws=s["ws"],
                                  stream=self._side)
        self._done[b].record(self._side)
        return s["residues"], s["k"]

    def done_event(self, slot: int):
        return self._done[slot]

    def drain(self, stream=None):
        """Make ``stream`` (default: the current one) wait for every outstanding step."""
        import torch
        cs = stream if stream is not None and hasattr(stream, "cuda_stream") else torch.cuda.current_stream()
        for e in self._done:
            cs.wait_event(e)
