"""GPU parity of the wide planner (plan_wide.cu: thread-block-cluster step
loop for N > 32 simulated nodes / global batch > 16384) against the oracle.

BASELINE cfg5 sweeps 32-256 logical ranks over a 1,048,576-id space; the
shapes here keep that rank count and per-rank batch structure at sizes the
oracle replays in seconds. LSG_PLAN_WIDE=1 also forces the wide path for
small worlds so both step-loop kernels face the same random configs.
"""
import os
import random

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import check_plan, u32

pytestmark = pytest.mark.gpu


@pytest.fixture
def force_wide():
    old = os.environ.get("LSG_PLAN_WIDE")
    os.environ["LSG_PLAN_WIDE"] = "1"
    yield
    if old is None:
        del os.environ["LSG_PLAN_WIDE"]
    else:
        os.environ["LSG_PLAN_WIDE"] = old


def replay_check(ls, out, ref, c):
    sim = ls.simulate_plan(out.plan, c.buffer_capacity)
    h, m = O.simulate(ref.items, ref.node_off, c.num_nodes, c.dataset_size, c.buffer_capacity)
    assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m), "replay"


@pytest.mark.parametrize("seed", range(30))
def test_wide_forced_random(ls, force_wide, seed):
    """The wide kernel on the same random family as the N <= 32 kernel."""
    r = random.Random(5000 + seed)
    N, b = r.choice([1, 2, 3, 4, 8, 16, 32]), r.choice([1, 2, 3, 5, 8, 16])
    B = N * b
    D = B * r.randint(1, 30) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 8), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([1, 2, 4, 8]))),
              drop_last=r.random() < 0.7, graph_mode=r.choice(["global", "pernode"]),
              optim_order=r.random() < 0.8, optim_remap=r.random() < 0.85,
              optim_balance=r.random() < 0.85, pso_iters=r.choice([10, 50]))
    check_plan(ls, c)


@pytest.mark.parametrize("seed", range(16))
def test_wide_many_nodes_random(ls, seed):
    """N in (32, 256]: multi-word holder masks, many balance donors."""
    r = random.Random(7000 + seed)
    N = r.choice([33, 40, 64, 100, 128, 200, 256])
    b = r.choice([1, 2, 4, 8, 16])
    B = N * b
    D = B * r.randint(1, 12) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 5), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, 2 * D // N)),
              drop_last=r.random() < 0.7, graph_mode=r.choice(["global", "pernode"]),
              optim_order=r.random() < 0.5, optim_remap=r.random() < 0.85,
              optim_balance=r.random() < 0.85, pso_iters=10)
    out, ref = check_plan(ls, c)
    replay_check(ls, out, ref, c)


@pytest.mark.parametrize("N", [32, 64, 128, 256])
def test_wide_cfg5_rank_sweep_shape(ls, N):
    """cfg5's structure (pooled buffer 50%, b=512) at a 65,536-id space:
    global batch N*512 (16,384 .. 131,072) and C = D / (2N)."""
    D = 1 << 16 if N <= 64 else N * 512 * 2
    c = O.Cfg(D, 3, N, 512, seed=42, buffer_capacity=D // (2 * N), optim_order=False)
    os.environ["LSG_PLAN_WIDE"] = "1"
    try:
        out, ref = check_plan(ls, c)
    finally:
        del os.environ["LSG_PLAN_WIDE"]
    replay_check(ls, out, ref, c)


def test_wide_cluster_sizes_agree(ls, force_wide):
    """The cluster width only partitions work: 1, 2, 4, 8 and 16 CTAs give
    the same plan."""
    c = O.Cfg(12000, 3, 48, 16, seed=11, buffer_capacity=300)
    ref = O.plan(c)
    old = os.environ.get("LSG_WIDE_CLUSTER")
    try:
        for p in ("1", "2", "4", "8", "16"):
            os.environ["LSG_WIDE_CLUSTER"] = p
            check_plan(ls, c, ref)
    finally:
        if old is None:
            os.environ.pop("LSG_WIDE_CLUSTER", None)
        else:
            os.environ["LSG_WIDE_CLUSTER"] = old


def test_wide_demo_and_goldens(ls, force_wide):
    """README demo through the wide kernel (proj/README.md:87)."""
    c = O.Cfg(1024, 6, 4, 8, seed=7, buffer_capacity=64)
    out, ref = check_plan(ls, c)
    sim = ls.simulate_plan(out.plan, 64)
    assert (sim.total_misses, sim.total_hits) == (4864, 1280)


def test_wide_properties_full_cfg5_slice(ls):
    """Full-size cfg5 index space (1,048,576 ids, 256 ranks, b=512), one
    epoch: size-independent invariants (every step's lists are a
    permutation of its global batch; fetch counts match the tags; balanced
    fetch spread <= 1)."""
    D, N, b = 1 << 20, 256, 512
    pc_ = O.Cfg(D, 2, N, b, seed=42, buffer_capacity=D // (2 * N), optim_order=False)
    from test_gpu_parity import to_pc
    out = ls.plan_schedule(to_pc(ls, pc_))
    tr = u32(out.trace.epochs)
    items = u32(out.plan.items)
    off = u32(out.plan.node_off)
    fa = u32(out.plan.fetches_after)
    B, S = N * b, D // (N * b)
    base = 0
    for g in range(2 * S):
        e, t = g // S, g % S
        step = items[base:base + off[g, N]]
        want = np.sort(tr[e, t * B:(t + 1) * B])
        assert np.array_equal(np.sort(step & 0x7FFFFFFF), want)
        fetch = (step >> 31) == 0
        cnt = np.array([int(fetch[off[g, k]:off[g, k + 1]].sum()) for k in range(N)])
        assert np.array_equal(cnt, fa[g])
        assert fa[g].max() - fa[g].min() <= 1
        base += off[g, N]


@pytest.mark.parametrize("seed", range(16))
def test_insert_redundant_planner(ls, seed):
    """chunk_insert_redundant (pipeline.cpp:103-114): after each step, the
    unrequested ids inside every node's chunk reads are inserted silently
    (buffer.cpp:48-53) with their next scheduled step — clairvoyant policy."""
    r = random.Random(8000 + seed)
    N, b = r.choice([1, 2, 4, 8, 40]), r.choice([2, 4, 8, 16])
    B = N * b
    D = B * r.randint(2, 16) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 6), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([2, 4, 8]))),
              drop_last=r.random() < 0.7, optim_order=r.random() < 0.6, optim_remap=r.random() < 0.8,
              optim_balance=r.random() < 0.8, optim_chunk=True, chunk_insert_redundant=True,
              chunk_threshold=r.choice([2, 5, 15, 40]), pso_iters=10)
    check_plan(ls, c)


@pytest.mark.parametrize("seed", range(10))
def test_insert_redundant_lru_planner_vs_reference(ls, seed):
    """plan_schedule with the LRU policy and chunk_insert_redundant
    (pipeline.cpp:103-114, LruBuffer::insert_silent = touch_or_insert): the
    plan file, metrics.csv and cost totals are byte-identical to the
    compiled reference's."""
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    from test_gpu_parity import to_pc
    r = random.Random(9300 + seed)
    N, b = r.choice([1, 2, 3, 4, 8]), r.choice([2, 4, 8, 16])
    B = N * b
    D = B * r.randint(2, 10) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 4), N, b, seed=r.randint(0, 10**6), buffer_capacity=r.randint(1, max(1, D // 3)),
              policy="lru", optim_chunk=True, chunk_insert_redundant=True, chunk_threshold=r.choice([2, 5, 15, 40]),
              optim_remap=r.random() < 0.8, optim_balance=r.random() < 0.8, pso_iters=10,
              drop_last=r.random() < 0.7)
    out = ls.plan_schedule(to_pc(ls, c))
    txt = O.ref_text(c)
    assert ls.format_plan(out.plan) == txt["plan"]
    sim = ls.simulate_plan(out.plan, c.buffer_capacity, "lru", insert_redundant=True)
    assert ls.format_metrics(out.plan, sim, "lru") == txt["metrics"]


@pytest.mark.parametrize("seed", range(12))
def test_insert_redundant_replay(ls, seed):
    """simulate_plan(..., insert_redundant=true) (buffer.cpp:224-238) on plans
    with and without redundant planning, vs the oracle (pinned to the
    reference in tests/test_oracle.py)."""
    r = random.Random(8500 + seed)
    N, b = r.choice([1, 2, 4, 8]), r.choice([2, 4, 8, 64])
    B = N * b
    D = B * r.randint(2, 12) + r.randint(0, B - 1)
    thr = r.choice([2, 5, 15, 40])
    c = O.Cfg(D, r.randint(1, 5), N, b, seed=r.randint(0, 10**6),
              buffer_capacity=r.randint(1, max(1, D // r.choice([2, 4, 8]))), optim_chunk=True,
              chunk_insert_redundant=r.random() < 0.5, chunk_threshold=thr, pso_iters=10)
    out, ref = check_plan(ls, c)
    sim = ls.simulate_plan(out.plan, c.buffer_capacity, insert_redundant=True)
    rs, re_, cnt, _, _ = O.plan_reads(ref.items, ref.node_off, N, True, thr)
    h, m = O.simulate_redundant(ref.items, ref.node_off, N, D, c.buffer_capacity, rs, re_, cnt)
    assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m)


@pytest.mark.parametrize("seed", range(8))
def test_insert_redundant_replay_lru_vs_reference(ls, seed):
    """simulate_plan(plan, C, Lru, insert_redundant=true): the silent inserts
    are LruBuffer::touch_or_insert (buffer.cpp:88-91) after each list. The
    plan is the REFERENCE's own LRU + chunk_insert_redundant plan (read from
    its plan file), and the rows must equal its metrics.csv hits/misses."""
    if not O.ref_available():
        pytest.skip("compiled reference not built")
    r = random.Random(9100 + seed)
    N, b = r.choice([1, 2, 4]), r.choice([2, 4, 8, 16])
    B = N * b
    D = B * r.randint(2, 10) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 4), N, b, seed=r.randint(0, 10**6), buffer_capacity=r.randint(1, max(1, D // 3)),
              policy="lru", optim_chunk=True, chunk_insert_redundant=True, chunk_threshold=r.choice([2, 5, 15]),
              pso_iters=10, drop_last=r.random() < 0.7)
    txt = O.ref_text(c)
    plan = ls.read_plan(txt["plan"])
    sim = ls.simulate_plan(plan, c.buffer_capacity, "lru", insert_redundant=True)
    rows = [ln.split(",") for ln in txt["metrics"].decode().splitlines()[1:]]
    T, N2 = plan.node_off.shape[0], plan.num_nodes
    want_h = np.array([int(x[3]) for x in rows], dtype=np.uint32).reshape(T, N2)
    want_m = np.array([int(x[4]) for x in rows], dtype=np.uint32).reshape(T, N2)
    assert np.array_equal(u32(sim.hits), want_h) and np.array_equal(u32(sim.misses), want_m)
    # and the oracle restatement agrees on the same plan
    rs, re_, cnt = u32(plan.read_start), u32(plan.read_end), u32(plan.read_count)
    h, m = O.simulate_redundant(u32(plan.items), u32(plan.node_off), N2, D, c.buffer_capacity, rs, re_, cnt, "lru")
    assert np.array_equal(h, want_h) and np.array_equal(m, want_m)
