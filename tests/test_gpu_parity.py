"""GPU parity: the sm_100a path (through the C ABI) vs the oracle.

The oracle is the C restatement (oracle/solar_oracle.c), itself pinned to the
compiled reference (tests/test_oracle.py). Everything here is bit-exact
integer work, so every comparison is array equality.
"""
import random

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


def u32(t):
    return t.detach().cpu().numpy().view(np.uint32)


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def to_pc(ls, c: O.Cfg):
    return ls.PipelineConfig(
        trace=ls.TraceConfig(c.dataset_size, c.num_epochs, c.num_nodes, c.local_batch, c.seed,
                             c.drop_last),
        buffer_capacity=c.buffer_capacity, policy=c.policy, graph_mode=c.graph_mode,
        chunk_threshold=c.chunk_threshold, chunk_insert_redundant=c.chunk_insert_redundant,
        pso=ls.PsoParams(c.pso_swarm, c.pso_iters, c.pso_p_personal, c.pso_p_global,
                         c.pso_inertia, c.pso_kick, c.pso_stagnation, c.pso_restart, c.seed),
        optim_order=c.optim_order, optim_remap=c.optim_remap, optim_balance=c.optim_balance,
        optim_chunk=c.optim_chunk)


# ------------------------------------------------------------------ K1 ---
def test_trace_goldens(ls):
    t = ls.generate_trace(ls.TraceConfig(8, 2, 2, 2, 42, True))
    assert u32(t.epochs).tolist() == [[7, 4, 1, 2, 5, 6, 0, 3], [0, 5, 2, 6, 4, 1, 7, 3]]
    t = ls.generate_trace(ls.TraceConfig(6, 2, 2, 1, 42, True))
    assert u32(t.epochs).tolist() == [[2, 4, 5, 0, 3, 1], [0, 4, 1, 5, 2, 3]]
    t = ls.generate_trace(ls.TraceConfig(1, 3, 1, 1, 5, True))
    assert u32(t.epochs).tolist() == [[0], [0], [0]]


@pytest.mark.parametrize("D,E,N,b,seed,dl", [
    (7, 1, 2, 2, 3, True), (7, 1, 2, 2, 3, False), (100, 3, 3, 7, 9, False),
    (16384, 10, 4, 64, 42, True), (262144, 3, 8, 512, 42, True), (131072, 4, 8, 64, 7, True),
    (1 << 20, 2, 32, 512, 42, True), (99991, 5, 3, 13, 1234567, False)])
def test_trace_matches_oracle(ls, D, E, N, b, seed, dl):
    got = u32(ls.generate_trace(ls.TraceConfig(D, E, N, b, seed, dl)).epochs)
    want = O.generate_trace(D, E, N, b, seed, dl)
    assert np.array_equal(got, want)


def test_trace_errors(ls):
    for cfg in [(3, 1, 2, 2, 0, True), (0, 1, 1, 1, 0, True), (4, 0, 1, 1, 0, True),
                (4, 1, 0, 1, 0, True), (4, 1, 1, 0, 0, True)]:
        with pytest.raises(ls.ConfigError):
            ls.generate_trace(ls.TraceConfig(*cfg))


# ------------------------------------------------------------------ K2/K3 ---
def test_graph_goldens(ls):
    t = ls.generate_trace(ls.TraceConfig(6, 3, 1, 2, 42, True))
    g = ls.build_reuse_graph(t, 3, "global")
    want = O.build_reuse_graph(u32(t.epochs), 6, 1, 2, 3, "global")
    assert u64(g.weights).ravel().tolist() == want.ravel().tolist()
    t2 = ls.generate_trace(ls.TraceConfig(6, 2, 2, 1, 42, True))
    gg = u64(ls.build_reuse_graph(t2, 2, "global").weights)
    gp = u64(ls.build_reuse_graph(t2, 2, "pernode").weights)
    assert gg[0, 1] == 1 and gg[1, 0] == 2 and gp[0, 1] == 4 and gp[1, 0] == 3


@pytest.mark.parametrize("seed", range(12))
def test_graph_matches_oracle_random(ls, seed):
    r = random.Random(seed)
    N, b = r.choice([1, 2, 3, 4, 8]), r.choice([1, 2, 5, 16])
    B = N * b
    D = B * r.randint(1, 40) + r.randint(0, B - 1)
    E = r.randint(1, 70)
    dl = r.random() < 0.6
    C = r.randint(1, max(1, D // N))
    mode = r.choice(["global", "pernode"])
    t = ls.generate_trace(ls.TraceConfig(D, E, N, b, seed, dl))
    got = u64(ls.build_reuse_graph(t, C, mode).weights)
    want = O.build_reuse_graph(u32(t.epochs), D, N, b, C, mode, dl)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", range(6))
def test_graph_general_trace_with_repeats(ls, seed):
    """read_trace admits repeated ids: windows count DISTINCT ids."""
    import torch
    r = np.random.default_rng(seed)
    N, b, E = 2, 3, 5
    D = 60
    ids = r.integers(0, D // 3, size=(E, 60)).astype(np.uint32)  # many repeats
    cfg = ls.TraceConfig(D, E, N, b, 0, True)
    t = ls.AccessTrace(cfg, torch.from_numpy(ids.view(np.int32)).cuda())
    for mode in ("global", "pernode"):
        for C in (1, 2, 5, 13):
            got = u64(ls.build_reuse_graph(t, C, mode).weights)
            want = O.build_reuse_graph(ids, D, N, b, C, mode, True)
            assert np.array_equal(got, want), (mode, C)


def test_graph_large_pernode(ls):
    D, E, N, b = 65536, 20, 8, 64
    t = ls.generate_trace(ls.TraceConfig(D, E, N, b, 3, True))
    for mode, C in (("global", 3000), ("pernode", 2000)):
        got = u64(ls.build_reuse_graph(t, C, mode).weights)
        want = O.build_reuse_graph(u32(t.epochs), D, N, b, C, mode, True)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("E,world", [(1, 1), (5, 2), (70, 3), (500, 8), (100, 7)])
def test_graph_row_blocks(ls, E, world):
    """lsg_build_reuse_graph_rows (the multi-GPU row sharding of K3): the row
    blocks of every rank_range split concatenate to build_reuse_graph."""
    import torch
    from paper_2211_00224_b200.parallel import rank_range
    D, N, b = 4096 if E <= 100 else 16384, 4, 8
    t = ls.generate_trace(ls.TraceConfig(D, E, N, b, E, True))
    for mode, C in (("global", D // 10), ("pernode", D // 12)):
        full = u64(ls.build_reuse_graph(t, C, mode).weights)
        parts = []
        for r in range(world):
            u0, u1 = rank_range(E, world, r)
            rows = ls.build_reuse_graph_rows(t, C, mode, u0, u1)
            parts.append(u64(rows))
        assert np.array_equal(np.concatenate(parts, axis=0), full), mode
    with pytest.raises(ls.ValidationError):
        ls.build_reuse_graph_rows(t, 10, "global", 0, E + 1)


# ------------------------------------------------------------------ K4 ---
@pytest.mark.parametrize("seed,E", [(s, E) for s, E in zip(range(14), [1, 2, 3, 5, 8, 10, 16, 31, 32, 33, 40, 64, 100, 200])])
def test_pso_matches_oracle(ls, seed, E):
    import torch
    r = np.random.default_rng(seed)
    w = r.integers(0, 1000, size=(E, E)).astype(np.uint64)
    np.fill_diagonal(w, 0)
    g = ls.ReuseGraph(E, 1, "global", torch.from_numpy(w.view(np.int64)).cuda())
    iters = 300 if E <= 64 else 120
    res = ls.pso_order(g, ls.PsoParams(max_iters=iters, seed=seed * 7 + 1))
    order, cost, hist, n = O.pso_order(w, seed * 7 + 1, iters=iters)
    assert u32(res.best.order).tolist() == order.tolist()
    assert res.best.cost == cost and res.iterations == n
    assert u64(res.history).tolist() == hist.tolist()


@pytest.mark.parametrize("params", [
    dict(swarm_size=1), dict(swarm_size=5, restart_limit=0), dict(swarm_size=64, restart_limit=3),
    dict(kick=0.0), dict(kick=0.3, inertia=0.9), dict(p_personal=1.0, p_global=0.0),
    dict(stagnation_limit=1), dict(max_iters=1)])
def test_pso_param_variants(ls, params):
    import torch
    E = 12
    r = np.random.default_rng(5)
    w = r.integers(0, 50, size=(E, E)).astype(np.uint64)
    np.fill_diagonal(w, 0)
    p = ls.PsoParams(**{**dict(max_iters=200, seed=9), **params})
    res = ls.pso_order(ls.ReuseGraph(E, 1, "global", torch.from_numpy(w.view(np.int64)).cuda()), p)
    order, cost, hist, n = O.pso_order(w, p.seed, swarm=p.swarm_size, iters=p.max_iters,
                                       p_personal=p.p_personal, p_global=p.p_global,
                                       inertia=p.inertia, kick=p.kick,
                                       stagnation=p.stagnation_limit, restart=p.restart_limit)
    assert u32(res.best.order).tolist() == order.tolist() and res.best.cost == cost
    assert res.iterations == n and u64(res.history).tolist() == hist.tolist()


# ------------------------------------------------------------------ K5/K6 ---
def check_plan(ls, c: O.Cfg, ref=None):
    out = ls.plan_schedule(to_pc(ls, c))
    ref = ref or O.plan(c)
    assert np.array_equal(u32(out.trace.epochs), ref.trace), "trace"
    assert np.array_equal(u64(out.graph.weights), ref.graph), "graph"
    assert u32(out.plan.order.order).tolist() == ref.order.tolist(), "order"
    assert out.plan.order.cost == ref.cost, "cost"
    np.testing.assert_array_equal(u32(out.plan.node_off), ref.node_off, "node_off")
    np.testing.assert_array_equal(u32(out.plan.fetches_before), ref.fb, "fetches_before")
    np.testing.assert_array_equal(u32(out.plan.fetches_after), ref.fa, "fetches_after")
    np.testing.assert_array_equal(u32(out.plan.items), ref.items, "items")
    return out, ref


def test_plan_readme_demo(ls):
    c = O.Cfg(1024, 6, 4, 8, seed=7, buffer_capacity=64)
    out, ref = check_plan(ls, c)
    assert u32(out.plan.order.order).tolist() == [5, 2, 3, 0, 1, 4] and out.plan.order.cost == 939


@pytest.mark.parametrize("seed", range(40))
def test_plan_matches_oracle_random(ls, seed):
    r = random.Random(1000 + seed)
    N, b = r.choice([1, 2, 3, 4, 8, 16, 32]), r.choice([1, 2, 3, 5, 8, 16])
    B = N * b
    D = B * r.randint(1, 30) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 8), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([1, 2, 4, 8]))),
              drop_last=r.random() < 0.7, graph_mode=r.choice(["global", "pernode"]),
              optim_order=r.random() < 0.8, optim_remap=r.random() < 0.85,
              optim_balance=r.random() < 0.85, optim_chunk=r.random() < 0.5,
              pso_iters=r.choice([10, 100]))
    check_plan(ls, c)


@pytest.mark.parametrize("D,E,N,b,frac", [(16384, 10, 4, 64, 0.10), (65536, 6, 8, 64, 0.05),
                                          (32768, 4, 8, 512, 0.20)])
def test_plan_benchmark_shapes(ls, D, E, N, b, frac):
    c = O.Cfg(D, E, N, b, seed=42, buffer_capacity=int(frac * D))
    check_plan(ls, c)


def test_plan_errors(ls):
    with pytest.raises(ls.ConfigError):
        ls.plan_schedule(to_pc(ls, O.Cfg(64, 2, 2, 4, buffer_capacity=0)))
    with pytest.raises(ls.ConfigError):
        ls.plan_schedule(to_pc(ls, O.Cfg(4, 2, 2, 4, buffer_capacity=3)))


@pytest.mark.parametrize("seed", range(24))
def test_plan_overlapped_loop_forced(ls, seed):
    """The overlapped step loop (K6o: classify / resolve / advance pipelined
    over three steps, stamps for two pending batches, re-classification on a
    conflict) runs by default only for B >= 2048; LSG_PLAN_OV=1 forces it on
    small random shapes: 1-3 step jobs, ragged last batches (drop_last off),
    every N <= 8 (B % 4 == 0), tight and loose buffers."""
    import os
    r = random.Random(7000 + seed)
    while True:
        N, b = r.choice([1, 2, 3, 4, 5, 8]), r.choice([4, 8, 12, 16, 32, 64])
        if (N * b) % 4 == 0:
            break
    B = N * b
    D = B * r.choice([1, 2, 3, 7, 20]) + (r.randint(0, B - 1) if seed % 3 else 0)
    c = O.Cfg(D, r.randint(1, 7), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([1, 2, 4, 8]))),
              drop_last=r.random() < 0.5, graph_mode=r.choice(["global", "pernode"]),
              optim_order=r.random() < 0.8, optim_remap=True,
              optim_balance=r.random() < 0.85, optim_chunk=r.random() < 0.5, pso_iters=30)
    os.environ["LSG_PLAN_OV"] = "1"
    try:
        check_plan(ls, c)
    finally:
        del os.environ["LSG_PLAN_OV"]


@pytest.mark.parametrize("D,E,N,b,frac,seed", [(65536, 3, 32, 512, 0.5 / 32, 1), (40000, 4, 16, 1000, 0.03, 2),
                                               (32768 + 777, 3, 32, 300, 0.02, 3)])
@pytest.mark.parametrize("kernel", ["0", "1"])
def test_plan_large_global_batch(ls, D, E, N, b, frac, seed, kernel):
    """global batch > 8192 (cfg5's 32-rank shape, b=512 -> B=16384) through
    both step-loop kernels: the single-CTA one with per-item arrays in
    L2-resident global scratch (LSG_PLAN_WIDE=0) and the cluster one."""
    import os
    c = O.Cfg(D, E, N, b, seed=seed, buffer_capacity=max(1, int(frac * D)), pso_iters=30,
              drop_last=seed != 3)
    os.environ["LSG_PLAN_WIDE"] = kernel
    try:
        out, ref = check_plan(ls, c)
    finally:
        del os.environ["LSG_PLAN_WIDE"]
    sim = ls.simulate_plan(out.plan, c.buffer_capacity)
    h, m = O.simulate(ref.items, ref.node_off, N, D, c.buffer_capacity)
    assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m)


@pytest.mark.parametrize("seed", range(10))
def test_plan_reads_match_oracle(ls, seed):
    """StepPlan.reads: plan_chunks (chunking.cpp:9-33) or singles (pipeline.cpp:21-28)."""
    r = random.Random(3000 + seed)
    N, b = r.choice([1, 2, 4, 8]), r.choice([2, 4, 8, 32])
    D = N * b * r.randint(2, 12) + r.randint(0, N * b - 1)
    c = O.Cfg(D, r.randint(1, 5), N, b, seed=seed, buffer_capacity=r.randint(1, max(1, D // 3)),
              optim_chunk=r.random() < 0.7, chunk_threshold=r.randint(1, 60), drop_last=r.random() < 0.7,
              pso_iters=20)
    out, ref = check_plan(ls, c)
    rs, re_, cnt, need, red = O.plan_reads(ref.items, ref.node_off, N, c.optim_chunk, c.chunk_threshold)
    p = out.plan
    assert np.array_equal(u32(p.read_count), cnt) and np.array_equal(u32(p.read_needed), need)
    assert np.array_equal(u32(p.read_redundant), red)
    grs, gre = u32(p.read_start), u32(p.read_end)
    base = 0
    for g in range(ref.node_off.shape[0]):
        for k in range(N):
            lo, n = base + ref.node_off[g, k], cnt[g, k]
            assert np.array_equal(grs[lo:lo + n], rs[lo:lo + n]) and np.array_equal(gre[lo:lo + n], re_[lo:lo + n])
        base += ref.node_off[g, N]
