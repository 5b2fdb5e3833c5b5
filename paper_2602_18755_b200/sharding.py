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
* ``gather_tables``: config tables built for a rank's shard of windows
  (C3 / run_experiment planning), all-gathered as fixed-size rows (SURVEY.md
  §8e: "ncclAllGather of table slices").
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


def prefix_slice(n_cand: int, rank: int, world: int) -> tuple[int, int, int]:
    """rank's slice of one exhaustive decision as bs_slice's (digits, lo, hi):
    the assignments whose first `digits` digits (batch 0 most significant)
    form a number in [lo, hi).  One leading digit when there are at least as
    many rungs as ranks, else two; ranks beyond the |cand|^2 leading values
    get an empty slice.  Independent of the projection length, so ranks need
    not know K (bs_mpc_exhaustive_slice reads a shorter projection's missing
    digits as 0)."""
    digits = 1 if n_cand >= world else 2
    lo, hi = shard_bounds(n_cand ** digits, rank, world)
    return digits, lo, hi


def combine_slices(parts: list) -> tuple:
    """Single-process counterpart of argmin_over_ranks for one decision:
    parts = [(feasible, objective, code, feasible_count)] of a partition's
    slices; returns (objective, code, feasible_count) with objective/code
    None when no slice has a feasible assignment."""
    best = None
    count = 0
    for feasible, obj, code, n in parts:
        count += n
        if feasible:
            key = (_obj_bits(obj), code)
            if best is None or key < best:
                best = key
    if best is None:
        return None, None, count
    return struct.unpack("<d", struct.pack("<q", best[0]))[0], best[1], count


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


_ENTRY_FIELDS = 8  # phase, tp, freq bits, r_c bits, e_c bits (or -1), g_c, flags, k*
_ERRORS = ["", "latency model returned non-positive value", "power model returned non-positive value",
           "idle model: tp {tp} not present", "no completed request at R_c", "grid: unknown axis",
           "idle model: empty frequency set"]


def _bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


def _pack_entry(e) -> list:
    """flags: bit 0 saturated, bits 1.. the entry's error text (an index into
    the messages build_config_table can produce)."""
    kind = 0
    if e.error:
        kind = next((i for i, m in enumerate(_ERRORS) if i and m.format(tp=e.config.tp) == e.error), -1)
        if kind < 0:
            raise ValueError(f"gather_tables: unexpected entry error {e.error!r}")
    return [int(e.config.phase), int(e.config.tp), _bits(e.config.base_freq_mhz), _bits(e.r_c),
            _bits(e.e_c) if e.e_c is not None else -1, int(e.g_c), (1 if e.saturated else 0) | (kind << 1),
            int(e.k_star)]


def _unpack_entry(row):
    from . import pdsim as P

    f = lambda q: struct.unpack("<d", struct.pack("<q", int(q)))[0]  # noqa: E731
    phase, tp, fb, rb, eb, g, flags, ks = (int(x) for x in row)
    return P.ConfigTableEntry(P.InstanceConfig(P.Phase(phase), tp, f(fb)), f(rb), None if eb == -1 else f(eb), g,
                              bool(flags & 1), _ERRORS[flags >> 1].format(tp=tp), ks)


def gather_tables(local_tables: list, n_tables: int, group=None, device: str | torch.device = "cpu") -> list:
    """All-gather config tables built for this rank's shard
    (shard_bounds(n_tables, rank, world)) of n_tables windows; every table
    has the same candidate list.  Returns all n_tables tables in window
    order on every rank (every field, error text included, round-trips)."""
    n_cand = len(local_tables[0]) if local_tables else 0
    n_cand = int(max_over_ranks(float(n_cand), group, device))
    flat = [_pack_entry(e) for t in local_tables for e in t]
    rows = torch.tensor(flat, dtype=torch.int64, device=device).reshape(len(local_tables), n_cand * _ENTRY_FIELDS) \
        if flat else torch.zeros((0, n_cand * _ENTRY_FIELDS), dtype=torch.int64, device=device)
    allrows = gather_rows(rows, n_tables, group)
    return [[_unpack_entry(allrows[i, c * _ENTRY_FIELDS:(c + 1) * _ENTRY_FIELDS].tolist()) for c in range(n_cand)]
            for i in range(n_tables)]
