"""Host-side work partitioning for multi-GPU runs.

* Sequence-batch sharding: sequences are independent (no cross-sequence sharing, reading R27),
  so each rank owns whole sequences with its own pool, table and free list; `lpt_assign` balances
  ranks by a per-sequence cost (e.g. the Stage-1 pair count) with the longest-processing-time rule.
* KV-head sharding: `head_shard` gives each rank a contiguous slice of the KV heads; the
  per-(pair, layer) squared sums of the slices add up to the full ones (sum over heads), which is
  what memshare_block_distance PARTIAL -> all-reduce -> FINALIZE relies on.
"""
from __future__ import annotations

import heapq


def lpt_assign(costs, world: int):
    """Longest-processing-time-first assignment of items to `world` bins; returns
    a list of index lists (each ascending). Deterministic (ties -> lower index / lower rank)."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    heap = [(0, r) for r in range(world)]
    out = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        out[r].append(i)
        heapq.heappush(heap, (load + costs[i], r))
    return [sorted(x) for x in out]


def head_shard(num_kv_heads: int, world: int, rank: int):
    """(h_local, head_offset) of `rank`: heads split as evenly as possible (uneven splits allowed,
    e.g. Phi-4's 10 heads over 4 ranks -> 3, 3, 2, 2)."""
    base, extra = divmod(num_kv_heads, world)
    h_local = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return h_local, offset
