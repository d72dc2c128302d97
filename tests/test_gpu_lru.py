"""GPU parity of the LRU policy (LruBuffer, buffer.cpp:61-82) against the
oracle: the per-rank replay (simulate_plan with Policy::Lru), the planner
with policy=lru (plan_schedule advancing LRU buffers), and the baseline pass
(baseline_config, pipeline.cpp:122-131) including the README demo's
baseline 6109 misses (proj/README.md:87)."""
import random

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import check_plan, to_pc, u32

pytestmark = pytest.mark.gpu


def lru_replay_check(ls, plan, ref, c):
    sim = ls.simulate_plan(plan, c.buffer_capacity, "lru", want_slots=True)
    h, m = O.simulate(ref.items, ref.node_off, c.num_nodes, c.dataset_size, c.buffer_capacity, "lru")
    assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m), "lru replay"
    return sim


def test_readme_baseline_6109(ls):
    pc = ls.PipelineConfig(trace=ls.TraceConfig(1024, 6, 4, 8, 7, True), buffer_capacity=64)
    base = ls.baseline_config(pc)
    out = ls.plan_schedule(base)
    sim = ls.simulate_plan(out.plan, 64, "lru")
    assert sim.total_misses == 6109 and sim.total_hits == 6 * 1024 - 6109


@pytest.mark.parametrize("seed", range(24))
def test_lru_planner_and_replay_random(ls, seed):
    r = random.Random(9000 + seed)
    N, b = r.choice([1, 2, 3, 4, 8, 16, 40, 100]), r.choice([1, 2, 3, 5, 8, 16])
    B = N * b
    D = B * r.randint(1, 20) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 6), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([1, 2, 4, 8]))), policy="lru",
              drop_last=r.random() < 0.7, graph_mode=r.choice(["global", "pernode"]),
              optim_order=r.random() < 0.7, optim_remap=r.random() < 0.8,
              optim_balance=r.random() < 0.8, pso_iters=20)
    out, ref = check_plan(ls, c)
    lru_replay_check(ls, out.plan, ref, c)


@pytest.mark.parametrize("seed", range(8))
def test_lru_replay_of_clairvoyant_plans(ls, seed):
    """The LRU replay of a clairvoyant plan (the reference's policy pairing is
    free: simulate_plan takes any plan and any policy)."""
    r = random.Random(9500 + seed)
    N, b = r.choice([2, 4, 8]), r.choice([4, 8, 32])
    D = N * b * r.randint(4, 30)
    c = O.Cfg(D, r.randint(2, 6), N, b, seed=seed, buffer_capacity=r.randint(1, D // 2), pso_iters=20)
    out, ref = check_plan(ls, c)
    lru_replay_check(ls, out.plan, ref, c)


def test_lru_replay_foreign_plan_with_repeats(ls):
    """read_plan admits repeated ids inside one list (plan.cpp:85-214): LRU
    replays them exactly (the clairvoyant replay rejects them)."""
    import torch
    r = np.random.default_rng(3)
    N, D, T = 3, 40, 30
    lens = r.integers(0, 9, size=(T, N))
    node_off = np.zeros((T, N + 1), dtype=np.uint32)
    node_off[:, 1:] = np.cumsum(lens, axis=1)
    items = np.concatenate([r.integers(0, D // 2, size=int(l.sum())) for l in lens]).astype(np.uint32)
    plan = ls.SchedulePlan(D, N, 1, T, None, torch.from_numpy(items.view(np.int32)).cuda(),
                           torch.from_numpy(node_off.view(np.int32)).cuda(), None, None)
    for C in (1, 3, 7, 19):
        sim = ls.simulate_plan(plan, C, "lru")
        h, m = O.simulate(items, node_off, N, D, C, "lru")
        assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m), C


@pytest.mark.parametrize("D,E,N,b,frac", [(16384, 6, 4, 64, 0.10), (65536, 3, 8, 512, 0.20),
                                          (65536, 3, 64, 64, 0.01)])
def test_lru_benchmark_shapes(ls, D, E, N, b, frac):
    c = O.Cfg(D, E, N, b, seed=42, buffer_capacity=int(frac * D), policy="lru", pso_iters=30)
    out, ref = check_plan(ls, c)
    lru_replay_check(ls, out.plan, ref, c)
    base = O.Cfg(D, E, N, b, seed=42, buffer_capacity=int(frac * D), policy="lru", optim_order=False,
                 optim_remap=False, optim_balance=False, optim_chunk=False)
    bout, bref = check_plan(ls, base)
    lru_replay_check(ls, bout.plan, bref, base)


def test_lru_slots_are_a_valid_buffer_layout(ls):
    """Slots from the LRU replay: hits read the slot their id occupies, and at
    every step no two resident ids share a slot (< C)."""
    c = O.Cfg(4096, 4, 4, 32, seed=5, buffer_capacity=300, policy="lru", pso_iters=10)
    out = ls.plan_schedule(to_pc(ls, c))
    sim = ls.simulate_plan(out.plan, 300, "lru", want_slots=True)
    items = u32(out.plan.items) & 0x7FFFFFFF
    slots = u32(sim.slots)
    off = u32(out.plan.node_off)
    base = 0
    where = [dict() for _ in range(4)]
    for g in range(off.shape[0]):
        for k in range(4):
            for p in range(base + off[g, k], base + off[g, k + 1]):
                x, s = int(items[p]), int(slots[p])
                if s & 0x80000000:
                    assert where[k].get(x) == s & 0x7FFFFFFF
                elif s != 0xFFFFFFFE:
                    assert s < 300
                    for y in [y for y, t in where[k].items() if t == s]:
                        del where[k][y]
                    where[k][x] = s
        base += off[g, 4]
