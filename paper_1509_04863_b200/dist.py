"""Host-side multi-GPU logic (one process per GPU, torch.distributed).

* Batches of independent pairs shard with no data-path collective: rank r owns
  global pairs [r*B, (r+1)*B) (weak scaling) -- `pair_range`.
* One huge signal is split into contiguous, row-aligned chunks (rows of M1
  samples, so every chunk can use the packed fold kernel) -- `signal_chunks`;
  each rank folds its chunk with global-position semantics (tm_fold(offset,
  len)) and the partial folds are summed IN PLACE with ONE all-reduce of the
  flat y1 || y2 buffer -- `allreduce_folds` / `single.SingleSignal`.  The fold of Eq. 2 is
  additive over any partition of the positions (pinned in tests), so the sum
  is exactly the full fold.
* The correlation of that one signal can then be split by output blocks
  (SURVEY 8(e)(ii)): each rank runs tm_correlate_match_part for its part and the
  per-pair keys (order-preserving int64 of (max r, lowest k), include/tm.h) are
  combined with ONE all-reduce MAX -- `allreduce_max_keys`; tm_match_keys then
  gives identical residues and k on every rank.
No arithmetic of the method lives here.
"""
from __future__ import annotations


def pair_range(batch_per_rank: int, rank: int) -> tuple[int, int]:
    """Global pair indices [first, first + batch) owned by `rank`."""
    return rank * batch_per_rank, batch_per_rank


def signal_chunks(N: int, M1: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row-aligned chunks (offset, length) covering [0, N), one per rank.
    Rows (M1 samples) are dealt as evenly as possible; requires M1 | N."""
    if N % M1:
        raise ValueError("row-aligned chunks need M1 | N")
    rows = N // M1
    base, extra = divmod(rows, world)
    out, r0 = [], 0
    for r in range(world):
        nr = base + (1 if r < extra else 0)
        out.append((r0 * M1, nr * M1))
        r0 += nr
    return out


def allreduce_folds(y1, y2, group=None):
    """Sum partial folds across ranks IN PLACE (SUM over int32 or fp32): on return
    y1 and y2 themselves hold the full fold on every rank (they are also returned).
    When y1 and y2 are views of one contiguous buffer (``SingleSignal.flat``) that
    buffer is reduced with one collective and no copy; otherwise the two vectors
    are reduced one after the other."""
    import torch.distributed as dist
    base = y1.untyped_storage().data_ptr()
    same = (base == y2.untyped_storage().data_ptr() and y1.is_contiguous() and y2.is_contiguous())
    if same:
        import torch
        lo = min(y1.storage_offset(), y2.storage_offset())
        hi = max(y1.storage_offset() + y1.numel(), y2.storage_offset() + y2.numel())
        same = hi - lo <= y1.numel() + y2.numel() + 64   # only alignment padding in between
    if same:
        flat = torch.empty(0, dtype=y1.dtype, device=y1.device).set_(
            y1.untyped_storage(), lo, (hi - lo,), (1,))
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.all_reduce(y1, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(y2, op=dist.ReduceOp.SUM, group=group)
    return y1, y2


def allreduce_max_keys(keys, group=None):
    """Element-wise MAX of the split-correlation keys (int64 [batch][2]) over ranks."""
    import torch.distributed as dist
    dist.all_reduce(keys, op=dist.ReduceOp.MAX, group=group)
    return keys


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a per-rank timing across ranks (the slowest rank defines the step)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
