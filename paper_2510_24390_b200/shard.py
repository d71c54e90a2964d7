"""Multi-GPU plumbing for the expansion step: one process per GPU, no data-path collective.

The units of the hot path are independent queries (a query's branches only read
that query's prefix / point KV, §4 "Expansion"), so ranks never exchange KV, partials or
outputs.  Two launch modes:

* weak (default): every rank runs its own full batch of the configured workload (its own seed);
  per-GPU work is fixed as N grows.
* strong: the configured batch's queries are partitioned across ranks:
  contiguous equal blocks, query q -> rank floor(q * N / Q), when all queries cost the same;
  otherwise LPT greedy on each query's unique KV bytes, ties broken by query id.

The only collectives are the timing reductions after the timed region: max of the per-rank
device-timed milliseconds and sum of the branches processed (whole-job throughput).  They work
on any torch.distributed backend (nccl on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations


def partition_queries(costs, world: int) -> list[list[int]]:
    """Partition query ids 0..Q-1 over `world` ranks.  Equal costs: contiguous blocks
    floor(q*N/Q); otherwise LPT greedy (largest cost first onto the least-loaded rank, ties by
    query id / rank id).  Every query lands on exactly one rank; ids ascend within a rank."""
    if world < 1:
        raise ValueError(f"bad world {world}")
    costs = [float(c) for c in costs]
    n = len(costs)
    if n == 0 or all(c == costs[0] for c in costs):
        return [[q for q in range(n) if (q * world) // n == r] for r in range(world)]
    load = [0.0] * world
    parts = [[] for _ in range(world)]
    for q in sorted(range(n), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda i: (load[i], i))
        load[r] += costs[q]
        parts[r].append(q)
    return [sorted(p) for p in parts]


def rank_queries(n_queries: int, rank: int, world: int, scaling: str = "weak", costs=None) -> list[int]:
    """Query ids this rank expands.  weak: all of them (the rank's own batch, own seed);
    strong: this rank's block of partition_queries (costs default to equal)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if scaling not in ("weak", "strong"):
        raise ValueError(f"scaling must be 'weak' or 'strong', got {scaling!r}")
    if scaling == "weak" or world == 1:
        return list(range(n_queries))
    return partition_queries(costs if costs is not None else [1.0] * n_queries, world)[rank]


def rank_seed(base_seed: int, rank: int) -> int:
    """Seed of a rank's synthetic inputs (distinct per rank, identical across runs)."""
    return base_seed * 101 + rank


def reduce_timing(elapsed_ms: float, units: float, device=None) -> tuple[float, float]:
    """(max over ranks of elapsed_ms, sum over ranks of units).  Identity without an initialised
    process group or with one rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(elapsed_ms), float(units)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    u = torch.tensor([units], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())
