"""Multi-GPU plumbing for the loading path (one process per GPU).

The step recurrence (plan) is replicated on every GPU ("replicas only": it
couples all ranks' buffers at every one of the T dependent steps). Ranks'
replays and batch fetches are independent given the plan, so each GPU owns a
contiguous range of training ranks; the only collective is one all-reduce
that assembles the per-(step, rank) hit/miss rows (buffer.hpp:106-111 rows).
"""
from __future__ import annotations

import torch


def rank_range(num_ranks: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of training ranks [0, num_ranks) over `world`
    GPUs; GPU `rank` owns [k0, k1). Ranks never split across GPUs."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(num_ranks, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def combine_rows(hits: torch.Tensor, misses: torch.Tensor, group=None) -> None:
    """In-place: every GPU's [T, N] rows hold only its own ranks' columns
    (others zero); a SUM all-reduce yields the full SimResult rows everywhere."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hits, group=group)
        dist.all_reduce(misses, group=group)


def sharded_simulate(ls, plan, capacity: int, world: int, rank: int, want_slots: bool = False):
    """simulate_plan for this GPU's ranks, rows combined across GPUs."""
    k0, k1 = rank_range(plan.num_nodes, world, rank)
    sim = ls.simulate_plan(plan, capacity, node_range=(k0, k1), want_slots=want_slots)
    combine_rows(sim.hits, sim.misses)
    sim.total_hits = int(sim.hits.sum().item())
    sim.total_misses = int(sim.misses.sum().item())
    return sim, (k0, k1)
