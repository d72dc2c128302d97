"""CPU suite: pins the oracle (C restatement) to the reference's golden vectors
and known-answer tests, and — when oracle/_ref is built — to the compiled
reference itself on seeded configs. No GPU needed."""
import random

import numpy as np
import pytest

import oracle as O

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


# ---- prng (tests/test_prng.cpp:10-23, :33-42, :68-75)
def test_splitmix_goldens():
    assert O.splitmix_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    assert O.splitmix_stream(42, 2) == [0xBDD732262FEB6E95, 0x28EFE333B266F103]
    d = (O.splitmix_stream(1, 1)[0] >> 11) * (1.0 / 9007199254740992.0)
    assert abs(d - 0.5665615751722809) < 1e-15


# ---- trace (tests/test_trace.cpp:29-34; test_reuse_graph.cpp:47-49)
def test_trace_goldens():
    assert O.generate_trace(8, 2, 2, 2, 42).tolist() == [[7, 4, 1, 2, 5, 6, 0, 3], [0, 5, 2, 6, 4, 1, 7, 3]]
    assert O.generate_trace(6, 2, 2, 1, 42).tolist() == [[2, 4, 5, 0, 3, 1], [0, 4, 1, 5, 2, 3]]
    assert O.generate_trace(1, 3, 1, 1, 5).tolist() == [[0]] * 3
    t = O.generate_trace(7, 1, 2, 2, 3, drop_last=True)
    assert t.shape == (1, 4)
    t = O.generate_trace(7, 1, 2, 2, 3, drop_last=False)
    assert sorted(t[0].tolist()) == list(range(7))


def test_trace_config_errors():
    for cfg in [(3, 1, 2, 2, 0), (0, 1, 1, 1, 0), (4, 0, 1, 1, 0), (4, 1, 0, 1, 0), (4, 1, 1, 0, 0)]:
        with pytest.raises(O.OracleError) as e:
            O.generate_trace(*cfg)
        assert e.value.code == 2


# ---- reuse graph (tests/test_reuse_graph.cpp:87-104)
def test_graph_goldens():
    t = O.generate_trace(6, 3, 1, 2, 42)
    assert O.build_reuse_graph(t, 6, 1, 2, 3, "global").ravel().tolist() == [0, 1, 1, 1, 0, 2, 1, 2, 0]
    t2 = O.generate_trace(6, 2, 2, 1, 42)
    g = O.build_reuse_graph(t2, 6, 2, 1, 2, "global")
    p = O.build_reuse_graph(t2, 6, 2, 1, 2, "pernode")
    assert (g[0, 1], g[1, 0], p[0, 1], p[1, 0]) == (1, 2, 4, 3)


def test_graph_saturating_buffer_is_zero():
    t = O.generate_trace(64, 4, 2, 4, 9)
    assert not O.build_reuse_graph(t, 64, 2, 4, 32, "global").any()


# ---- epoch order (tests/test_epoch_order.cpp:69-86)
def test_brute_force_goldens():
    o, c = O.brute_force_order(np.array([[0, 9], [1, 0]], dtype=np.uint64))
    assert o.tolist() == [1, 0] and c == 1
    o, c = O.brute_force_order(np.full((4, 4), 5, dtype=np.uint64) * (1 - np.eye(4, dtype=np.uint64)))
    assert o.tolist() == [0, 1, 2, 3]
    ks = np.array([0, 2, 5, 1, 0, 3, 4, 2, 0], dtype=np.uint64).reshape(3, 3)
    o, c = O.brute_force_order(ks)
    assert o.tolist() == [2, 1, 0] and c == 3


def test_pso_properties():
    r = np.random.default_rng(1)
    for E in (3, 6, 9):
        w = r.integers(0, 100, size=(E, E)).astype(np.uint64)
        np.fill_diagonal(w, 0)
        o, c, h, n = O.pso_order(w, 5)
        ident = int(sum(w[i, i + 1] for i in range(E - 1)))
        _, best = O.brute_force_order(w)
        assert best <= c <= ident and sorted(o.tolist()) == list(range(E))
        assert all(h[i] >= h[i + 1] for i in range(len(h) - 1))


# ---- remap / balance worked examples (tests/test_locality.cpp, test_balance.cpp)
def _remap(buffers, batch, b, slice_=False):
    N = len(buffers)
    holders = [sum(1 << k for k in range(N) if x in buffers[k]) for x in batch]
    items, off = O.remap_step(holders, batch, N, b, slice_)
    return [[(int(v & 0x7FFFFFFF), bool(v >> 31)) for v in items[off[k]:off[k + 1]]] for k in range(N)]


def test_remap_worked_examples():
    assert _remap([{9}, {5, 7}], [5, 9, 2, 7], 2) == [[(9, True), (2, False)], [(5, True), (7, True)]]
    assert _remap([set(), set()], [5, 2, 7, 1], 2) == [[(5, False), (2, False)], [(7, False), (1, False)]]
    assert _remap([{1, 2, 3}, set()], [1, 2, 3, 9], 2) == [[(1, True), (2, True)], [(3, False), (9, False)]]
    assert _remap([{4, 8}, {4, 8}], [4, 8], 1) == [[(4, True)], [(8, True)]]
    assert _remap([{6, 4}, {4}], [6, 4], 2) == [[(6, True)], [(4, True)]]


def test_balance_worked_example():
    items = list(range(148))
    off = [0, 107, 148]
    it, off2, moves = O.balance_step(items, off)
    assert moves == 33 and list(off2) == [0, 74, 148]
    moved = it[off2[1] + 41:].tolist()
    assert moved[0] == 106 and moved[-1] == 74 and moved == sorted(moved, reverse=True)
    assert max(it[:74]) == 73


# ---- buffer (tests/test_buffer.cpp:11-27)
def test_buffer_worked_examples():
    assert O.simulate_sequence([0, 1, 0, 1], 1, "lru") == 4
    assert O.simulate_sequence([0, 1, 2, 0, 1], 2, "clairvoyant") == 3
    assert O.simulate_sequence([0, 1, 2, 0, 1], 2, "lru") == 5
    seq = [3, 1, 4, 1, 5, 9, 2, 6, 3, 1, 4, 5, 9, 2, 6]
    assert O.simulate_sequence(seq, 7, "lru") == 7 == O.simulate_sequence(seq, 7, "clairvoyant")


# ---- plan level (README.md:87,107-114; tests/test_pipeline.cpp:164-173)
def test_readme_demo():
    c = O.Cfg(1024, 6, 4, 8, seed=7, buffer_capacity=64)
    p = O.plan(c)
    h, m = O.simulate(p.items, p.node_off, 4, 1024, 64)
    assert (int(m.sum()), int(h.sum())) == (4864, 1280)
    assert p.order.tolist() == [5, 2, 3, 0, 1, 4] and p.cost == 939
    base = O.Cfg(1024, 6, 4, 8, seed=7, buffer_capacity=64, policy="lru", optim_order=False,
                 optim_remap=False, optim_balance=False, optim_chunk=False)
    pb = O.plan(base)
    hb, mb = O.simulate(pb.items, pb.node_off, 4, 1024, 64, "lru")
    assert int(mb.sum()) == 6109


def test_whole_dataset_buffer_only_cold_misses():
    c = O.Cfg(64, 3, 1, 8, seed=5, buffer_capacity=64)
    p = O.plan(c)
    h, m = O.simulate(p.items, p.node_off, 1, 64, 64)
    assert int(m.sum()) == 64 and int(h.sum()) == 3 * 64 - 64


# ---- store (tests/test_store.cpp:63-65)
def test_store_payload_golden():
    assert bytes(O.store_payload(1, 0, 32)).hex() == \
        "c15c0289ec2d0a9167ec8e65a18debbe5e5532fbeea293f80bc942ee9086c171"


# ---- restatement vs the compiled reference (oracle/_ref)
ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@ref
@pytest.mark.parametrize("seed", range(40))
def test_oracle_matches_reference(seed):
    r = random.Random(seed)
    N, b = r.choice([1, 2, 3, 4, 8]), r.choice([1, 2, 3, 5, 8])
    B = N * b
    D = B * r.randint(1, 12) + r.randint(0, B - 1)
    cfg = O.Cfg(D, r.randint(1, 8), N, b, seed=r.randint(0, 1000),
                buffer_capacity=r.randint(1, max(1, D // 2)), drop_last=r.random() < 0.7,
                policy=r.choice(["clairvoyant", "lru"]), graph_mode=r.choice(["global", "pernode"]),
                optim_order=r.random() < 0.8, optim_remap=r.random() < 0.8,
                optim_balance=r.random() < 0.8, optim_chunk=r.random() < 0.8,
                chunk_insert_redundant=r.random() < 0.3, chunk_threshold=r.randint(1, 6),
                pso_iters=r.choice([5, 50, 500]))
    p, q = O.plan(cfg, residency=True), O.ref_plan(cfg)
    for f in ("trace", "graph", "order", "items", "node_off", "fb", "fa", "hist"):
        assert np.array_equal(getattr(p, f), getattr(q, f)), f
    assert (p.cost, p.iters) == (q.cost, q.iters)
    if not (cfg.chunk_insert_redundant and cfg.optim_chunk):
        h, m = O.simulate(p.items, p.node_off, N, D, cfg.buffer_capacity, cfg.policy)
        assert np.array_equal(p.residency, q.residency)
        assert np.array_equal(h, q.hits) and np.array_equal(m, q.misses)
    else:  # the reference replays with insert_redundant too (pipeline.cpp:266-275)
        rs, re_, cnt, _, _ = O.plan_reads(p.items, p.node_off, N, True, cfg.chunk_threshold)
        h, m = O.simulate_redundant(p.items, p.node_off, N, D, cfg.buffer_capacity, rs, re_, cnt, cfg.policy)
        assert np.array_equal(h, q.hits) and np.array_equal(m, q.misses)


@ref
def test_oracle_matches_reference_config1():
    c = O.Cfg(16384, 10, 4, 64, seed=42, buffer_capacity=1638)
    p, q = O.plan(c), O.ref_plan(c)
    assert np.array_equal(p.items, q.items) and np.array_equal(p.node_off, q.node_off)
    h, m = O.simulate(p.items, p.node_off, 4, 16384, 1638)
    assert np.array_equal(m, q.misses)


@ref
def test_oracle_simulate_matches_reference_on_foreign_plans():
    """simulate_plan replays any plan file (tools/loadsched.cpp:154-184)."""
    r = np.random.default_rng(3)
    N, D, T = 3, 40, 12
    lens = r.integers(0, 6, size=(T, N))
    node_off = np.zeros((T, N + 1), dtype=np.uint32)
    node_off[:, 1:] = np.cumsum(lens, axis=1)
    items = np.concatenate([r.choice(D, size=int(l.sum()), replace=False) for l in lens]).astype(np.uint32)
    for C in (1, 3, 10):
        h, m = O.simulate(items, node_off, N, D, C)
        hr, mr = O.ref_simulate(items, node_off, N, D, 4, C)
        assert np.array_equal(h, hr) and np.array_equal(m, mr)


@ref
def test_store_payload_matches_reference():
    got = O.ref_store(5, 24, 77)
    assert np.array_equal(got, O.store_payload(77, 0, 120))


@ref
@pytest.mark.parametrize("seed", range(12))
def test_oracle_reads_match_reference(seed):
    """StepPlan::reads (chunking.cpp:9-33, pipeline.cpp:21-28, :83-88)."""
    r = random.Random(900 + seed)
    N, b = r.choice([1, 2, 4]), r.choice([2, 4, 8])
    D = N * b * r.randint(2, 10) + r.randint(0, N * b - 1)
    cfg = O.Cfg(D, r.randint(1, 4), N, b, seed=seed, buffer_capacity=r.randint(1, max(1, D // 3)),
                optim_chunk=r.random() < 0.7, chunk_threshold=r.randint(1, 40), pso_iters=20)
    p, q = O.plan(cfg), O.ref_plan(cfg)
    rs, re_, cnt, need, red = O.plan_reads(p.items, p.node_off, N, cfg.optim_chunk, cfg.chunk_threshold)
    assert np.array_equal(cnt.ravel(), q.extra["rcount"]) and np.array_equal(need.ravel(), q.extra["rneed"])
    assert np.array_equal(red.ravel(), q.extra["rred"])
    base = 0
    for g in range(p.node_off.shape[0]):
        for k in range(N):
            lo = base + p.node_off[g, k]
            n = cnt[g, k]
            assert np.array_equal(rs[lo:lo + n], q.extra["rstart"][lo:lo + n])
            assert np.array_equal(re_[lo:lo + n], q.extra["rend"][lo:lo + n])
        base += p.node_off[g, N]


@ref
@pytest.mark.parametrize("seed", range(6))
def test_oracle_matches_reference_many_nodes(seed):
    """N > 32 simulated ranks (cfg5's 32-256 logical-rank sweep) at small D."""
    r = random.Random(4200 + seed)
    N, b = r.choice([33, 64, 100, 256]), r.choice([1, 2, 4])
    B = N * b
    D = B * r.randint(1, 6) + r.randint(0, B - 1)
    cfg = O.Cfg(D, r.randint(1, 3), N, b, seed=r.randint(0, 1000),
                buffer_capacity=r.randint(1, max(1, 2 * D // N)), drop_last=r.random() < 0.7,
                optim_order=r.random() < 0.5, optim_remap=r.random() < 0.85,
                optim_balance=r.random() < 0.85, pso_iters=20)
    p, q = O.plan(cfg, residency=True), O.ref_plan(cfg)
    for f in ("trace", "items", "node_off", "fb", "fa"):
        assert np.array_equal(getattr(p, f), getattr(q, f)), f
    h, m = O.simulate(p.items, p.node_off, N, D, cfg.buffer_capacity)
    assert np.array_equal(p.residency, q.residency)
    assert np.array_equal(h, q.hits) and np.array_equal(m, q.misses)


def test_full_shape_goldens_hold_survey_anchors():
    """tests/golden/full_shapes.json (the reference's outputs at the full
    BASELINE shapes, tools/make_goldens.py) holds the figures SURVEY.md §6
    recorded from the compiled reference during the survey."""
    import json
    import os
    GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_shapes.json")))
    assert (GOLD["cfg2_global"]["total_hits"], GOLD["cfg2_global"]["total_misses"]) == (25870743, 343657)
    assert GOLD["cfg2_pernode"]["iterations"] == 444 and GOLD["cfg2_pernode"]["cost"] == 22682160
    assert GOLD["cfg4"]["cost"] == 15637500 and GOLD["cfg4"]["iterations"] == 500
    assert GOLD["cfg4"]["graph_sum"] == pytest.approx(7.85e9, rel=5e-3)
    assert GOLD["cfg1"]["iterations"] == 121 and GOLD["cfg1"]["cost"] == 34977
    assert (GOLD["cfg1"]["total_misses"], GOLD["cfg1"]["total_hits"]) == (104872, 58968)
