"""Multi-GPU partitioning of the decision path.

One process per GPU.  Every unit of the path is independent -- decisions,
snapshots, what-if scenarios, placement candidates -- so units are split into
contiguous per-rank shards with no data-path collective; the only exchange
is at the end:

* ``gather_rows``: the per-unit result rows of every rank, in global unit
  order (``all_gather`` of fixed-size rows; bytes per decision).
* ``argmin_over_ranks``: one decision whose code space is sliced by leading
  digits across ranks; the global (objective, code) minimum is two MIN
  all-reduces: first over the objective's bit pattern (objectives are
  non-negative doubles, whose IEEE bit patterns order like the values), then
  over the code among the ranks holding that objective (others contribute
  INT64_MAX).  This is the exhaustive-MPC tie rule (dvfs.hpp:243: smallest
  objective, then lexicographically smallest assignment = smallest code).
* ``max_over_ranks``: the timing rule of bench.py (max of per-rank device
  times).

The functions take a ``torch.distributed`` process group, so the same code
runs over NCCL on the GPU box and over gloo in the CPU tests.
"""
from __future__ import annotations

import struct

import torch
import torch.distributed as dist

INT64_MAX = (1 << 63) - 1


def shard_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n units for `rank` of `world`
    (the first n % world ranks take one extra unit)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("shard_bounds: bad rank/world/n")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def code_slice(n_cand: int, K: int, rank: int, world: int) -> tuple[int, int]:
    """Code range [lo, hi) of rank's slice of one decision's n_cand^K
    assignments, cut at leading-digit boundaries (batch 0 is the most
    significant digit) so each slice is a union of whole subtrees."""
    total = n_cand ** K
    lead = 1
    depth = 0
    while lead < world and depth < K:
        lead *= n_cand
        depth += 1
    sub = total // lead  # codes per leading prefix
    lo_p, hi_p = shard_bounds(lead, rank, world)
    return lo_p * sub, hi_p * sub


def _obj_bits(x: float) -> int:
    if not x >= 0.0:
        raise ValueError("argmin_over_ranks: objectives are non-negative")
    return struct.unpack("<q", struct.pack("<d", x))[0]


def argmin_over_ranks(objective: float | None, code: int | None, group=None,
                      device: str | torch.device = "cpu") -> tuple[float | None, int | None]:
    """Global (objective, code) minimum; a rank with nothing feasible passes
    None.  Returns (None, None) when no rank has a candidate."""
    bits = _obj_bits(objective) if objective is not None else INT64_MAX
    t = torch.tensor([bits], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    best_bits = int(t.item())
    if best_bits == INT64_MAX:
        return None, None
    c = torch.tensor([code if (objective is not None and bits == best_bits) else INT64_MAX], dtype=torch.int64,
                     device=device)
    dist.all_reduce(c, op=dist.ReduceOp.MIN, group=group)
    return struct.unpack("<d", struct.pack("<q", best_bits))[0], int(c.item())


def gather_rows(rows: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather per-unit rows (shape [n_local, w], any dtype) sharded by
    shard_bounds(n_total, rank, world); returns [n_total, w] in global order
    on every rank."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_bounds(n_total, rank, world)
    if rows.shape[0] != hi - lo:
        raise ValueError("gather_rows: local rows do not match this rank's shard")
    cap = -(-n_total // world)
    pad = torch.zeros((cap,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    pad[: rows.shape[0]] = rows
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    out = []
    for r in range(world):
        a, b = shard_bounds(n_total, r, world)
        out.append(parts[r][: b - a])
    return torch.cat(out, 0)


def max_over_ranks(value: float, group=None, device: str | torch.device = "cpu") -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
