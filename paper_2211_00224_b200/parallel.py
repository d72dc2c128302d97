"""Multi-GPU plumbing for the loading path (one process per GPU).

* K1 shuffle: every GPU generates all epochs (cheap; no exchange).
* K3 reuse matrix: rows shard. Every GPU builds all window bitsets and the
  row block [u0, u1) of w; one all-gather of the row blocks assembles
  build_reuse_graph's weights (reuse_graph.cpp:77-101) everywhere.
* K4 PSO and K6 step loop: replicas only (the step recurrence couples all
  ranks' buffers at every one of the T dependent steps); deterministic, so
  every GPU holds the identical plan.
* K7 replay / K8 fetch: each GPU owns a contiguous range of training ranks;
  one all-gather of the per-rank [T] hit/miss columns assembles SimResult's
  rows (buffer.hpp:106-111). The fetch moves no data between GPUs.
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


def _dist(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        return dist
    return None


def allgather_blocks(block: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather of contiguous row blocks split by rank_range(total, world):
    GPU r contributes rows [k0, k1) of a [total, ...] tensor (`block`, shape
    [k1 - k0, ...]); returns the full tensor on every GPU. Blocks are padded to
    the largest span so one equal-size all-gather (NCCL over NVLink, or gloo)
    moves them."""
    dist = _dist(group)
    if dist is None:
        return block
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    spans = [rank_range(total, world, r) for r in range(world)]
    k0, k1 = spans[rank]
    if block.shape[0] != k1 - k0:
        raise ValueError("block rows do not match this GPU's rank_range span")
    span = max(b - a for a, b in spans)
    pad = block.new_zeros((span,) + tuple(block.shape[1:]))
    pad[: k1 - k0] = block
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: b - a] for p, (a, b) in zip(parts, spans)], dim=0)


def combine_rows(hits: torch.Tensor, misses: torch.Tensor, group=None) -> None:
    """In-place: every GPU's [T, N] rows hold valid values only in its own
    ranks' columns [k0, k1); one all-gather of the stacked per-rank [T] hit
    and miss columns yields the full SimResult rows on every GPU."""
    dist = _dist(group)
    if dist is None:
        return
    N = hits.shape[1]
    k0, k1 = rank_range(N, dist.get_world_size(group), dist.get_rank(group))
    mine = torch.stack([hits[:, k0:k1].t(), misses[:, k0:k1].t()], dim=1).contiguous()  # [k, 2, T]
    full = allgather_blocks(mine, N, group)  # [N, 2, T]
    hits.copy_(full[:, 0].t())
    misses.copy_(full[:, 1].t())


def sharded_reuse_graph(ls, trace, buffer_size: int, mode: str = "global", group=None):
    """build_reuse_graph (reuse_graph.cpp:77-101) with the rows of w sharded
    over the GPUs of `group` (lsg_build_reuse_graph_rows) and all-gathered;
    identical to ls.build_reuse_graph on every GPU."""
    dist = _dist(group)
    if dist is None:
        return ls.build_reuse_graph(trace, buffer_size, mode)
    E = trace.epochs.shape[0]
    u0, u1 = rank_range(E, dist.get_world_size(group), dist.get_rank(group))
    rows = ls.build_reuse_graph_rows(trace, buffer_size, mode, u0, u1)
    w = allgather_blocks(rows, E, group)
    return ls.ReuseGraph(E, buffer_size, mode, w)


def sharded_simulate(ls, plan, capacity: int, world: int, rank: int, want_slots: bool = False):
    """simulate_plan for this GPU's ranks, rows combined across GPUs."""
    k0, k1 = rank_range(plan.num_nodes, world, rank)
    sim = ls.simulate_plan(plan, capacity, node_range=(k0, k1), want_slots=want_slots)
    combine_rows(sim.hits, sim.misses)
    sim.total_hits = int(sim.hits.sum().item())
    sim.total_misses = int(sim.misses.sum().item())
    return sim, (k0, k1)
