"""GPU parity of the per-call entry points against the oracle: remap_step /
slice_step (locality.cpp:7-73) against explicit residency sets, balance_step
(balance.cpp:10-39), plan_chunks (chunking.cpp:9-33), brute_force_order
(epoch_order.cpp:32-52), the Buffer object, simulate_sequence and
optimal_miss_oracle (buffer.cpp:10-182). The same device code runs inside the planner's
step loop; these calls expose it one step at a time, like the reference's
own test_locality / test_balance suites use it."""
import random

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

HIT = 0x80000000


def holders_of(buffers, batch):
    return [sum(1 << k for k, s in enumerate(buffers) if x in s) for x in batch]


def py_remap(buffers, batch, b):
    """locality.cpp:7-39 as plain loops (for N > 64, beyond the C oracle)."""
    N = len(buffers)
    nodes = [[] for _ in range(N)]
    fetches = []
    for x in batch:
        ch = None
        for k in range(N):
            if len(nodes[k]) >= b or x not in buffers[k]:
                continue
            if ch is None or len(nodes[k]) < len(nodes[ch]):
                ch = k
        if ch is None:
            fetches.append(x)
        else:
            nodes[ch].append(x | HIT)
    k = 0
    for x in fetches:
        while len(nodes[k]) >= b:
            k += 1
        nodes[k].append(x)
    items = [v for n in nodes for v in n]
    off = np.cumsum([0] + [len(n) for n in nodes]).astype(np.uint32)
    return np.array(items, dtype=np.uint32), off


def rand_case(rng, N, b, D, fill, dup=False):
    length = rng.randint(0, N * b)
    batch = [rng.randrange(D) for _ in range(length)] if dup else rng.sample(range(D), min(length, D))
    buffers = [set(rng.sample(range(D), min(D, int(fill * D)))) for _ in range(N)]
    return buffers, batch


@pytest.mark.parametrize("slice_", [False, True])
@pytest.mark.parametrize("N", [1, 2, 3, 8, 33, 64])
def test_remap_and_slice_match_oracle(ls, N, slice_):
    rng = random.Random(N * 7 + slice_)
    for case in range(12):
        b = rng.choice([1, 2, 5, 16, 64])
        D = rng.choice([N * b, 4 * N * b, 1000])
        buffers, batch = rand_case(rng, N, b, D, rng.choice([0.0, 0.1, 0.5, 0.9]), dup=case % 3 == 2)
        fn = ls.slice_step if slice_ else ls.remap_step
        items, off = fn(buffers, batch, b)
        ri, ro = O.remap_step(holders_of(buffers, batch), batch, N, b, slice_)
        assert np.array_equal(off, ro), (N, b, case)
        assert np.array_equal(items, ri), (N, b, case)


def test_remap_many_nodes_matches_loops(ls):
    rng = random.Random(5)
    for N in (65, 128, 256):
        for _ in range(4):
            b = rng.choice([1, 3, 8])
            buffers, batch = rand_case(rng, N, b, 3 * N * b, rng.choice([0.05, 0.3]))
            items, off = ls.remap_step(buffers, batch, b)
            ri, ro = py_remap(buffers, batch, b)
            assert np.array_equal(off, ro) and np.array_equal(items, ri), (N, b)


def test_remap_validation(ls):
    with pytest.raises(ls.ValidationError, match="remap_step: no nodes"):
        ls.remap_step([], [1], 1)
    with pytest.raises(ls.ValidationError, match="local_batch must be >= 1"):
        ls.remap_step([set()], [1], 0)
    with pytest.raises(ls.ValidationError, match="batch larger than N \\* local_batch"):
        ls.remap_step([set(), set()], [1, 2, 3], 1)
    with pytest.raises(ls.ValidationError, match="slice_step: no nodes"):
        ls.slice_step([], [1], 1)
    items, off = ls.remap_step([set(), set()], [], 4)
    assert items.size == 0 and list(off) == [0, 0, 0]


def rand_lists(rng, N, maxlen, hit_p):
    items, off = [], [0]
    for _ in range(N):
        n = rng.randint(0, maxlen)
        for _ in range(n):
            x = rng.randrange(1 << 20)
            items.append(x | (HIT if rng.random() < hit_p else 0))
        off.append(len(items))
    return np.array(items, dtype=np.uint32), np.array(off, dtype=np.uint32)


@pytest.mark.parametrize("N", [1, 2, 5, 32, 100, 256])
def test_balance_matches_oracle(ls, N):
    rng = random.Random(N)
    for case in range(10):
        items, off = rand_lists(rng, N, rng.choice([3, 40, 300]), rng.choice([0.0, 0.3, 0.8]))
        if case % 4 == 3 and items.size:  # duplicate ids inside one donor
            items[off[0]:off[1]] = items[off[0]] & ~np.uint32(HIT)
        gi, go, gm = ls.balance_step(items, off)
        ri, ro, rm = O.balance_step(items, off)
        assert gm == rm and np.array_equal(go, ro) and np.array_equal(gi, ri), (N, case)


def test_balance_wide_spread_uses_the_round_simulation(ls):
    # one node with 5000 fetches, the rest empty: > 2048 count levels
    for N in (2, 7, 64):
        items = np.arange(5000, dtype=np.uint32)[::-1].copy()
        off = np.array([0] + [5000] * N, dtype=np.uint32)
        gi, go, gm = ls.balance_step(items, off)
        ri, ro, rm = O.balance_step(items, off)
        assert gm == rm and np.array_equal(go, ro) and np.array_equal(gi, ri), N


def test_balance_no_nodes(ls):
    with pytest.raises(ls.ValidationError, match="balance_step: no nodes"):
        ls.balance_step([], [0])


def test_plan_chunks_matches_oracle(ls):
    rng = random.Random(3)
    for thr in (1, 2, 15, 100):
        for n in (0, 1, 7, 300, 5000):
            ids = [rng.randrange(20000) for _ in range(n)]
            cp = ls.plan_chunks(ids, thr)
            rs, re_, cnt, need, red = O.plan_reads(np.array(ids, np.uint32), np.array([0, n], np.uint32), 1,
                                                   True, thr)
            got = [(r.start, r.end) for r in cp.reads]
            assert got == list(zip(rs[: cnt[0, 0]].tolist(), re_[: cnt[0, 0]].tolist())), (thr, n)
            assert cp.needed == need[0, 0] and cp.redundant == red[0, 0]
            assert all((r.kind == "single") == (r.start == r.end) for r in cp.reads)


def test_brute_force_matches_oracle(ls):
    import torch

    rng = np.random.default_rng(9)
    for E in (1, 2, 5, 8, 10):
        w = rng.integers(0, 6, size=(E, E)).astype(np.int64)  # small range: many ties
        g = ls.ReuseGraph(E, 1, "global", torch.from_numpy(w).cuda())
        o = ls.brute_force_order(g)
        ro, rc = O.brute_force_order(w.astype(np.uint64))
        assert o.cost == rc and o.order.cpu().numpy().tolist() == ro.tolist(), E


def next_use_chain(seq):
    nxt, last = [O_NEVER] * len(seq), {}
    for i in range(len(seq) - 1, -1, -1):
        nxt[i] = last.get(seq[i], O_NEVER)
        last[seq[i]] = i
    return nxt


O_NEVER = (1 << 64) - 1


@pytest.mark.parametrize("policy", ["clairvoyant", "lru"])
def test_simulate_sequence_and_buffer_match_oracle(ls, policy):
    rng = random.Random(11 if policy == "lru" else 12)
    for _ in range(12):
        n = rng.choice([1, 17, 300, 3000])
        ids = rng.choice([3, 50, 1000])
        C = rng.choice([1, 2, 7, 64, 500])
        seq = [rng.randrange(ids) for _ in range(n)]
        want = O.simulate_sequence(seq, C, policy)
        assert ls.simulate_sequence(seq, C, policy) == want, (n, ids, C)
        buf = ls.make_buffer(policy, C)
        hits = buf.access_batch(seq, next_use_chain(seq))
        assert int((~hits).sum()) == want, (n, ids, C)
        assert len(buf.resident()) == min(C, len(set(seq))) or policy == "clairvoyant"


def test_buffer_worked_examples(ls):
    buf = ls.make_buffer("lru", 2)
    buf.insert_silent(5)
    assert 5 in buf.resident() and buf.access(5) and not buf.access(6) and len(buf.resident()) == 2
    cv = ls.make_buffer("clairvoyant", 2)
    for x in (0, 1, 2):
        cv.access(x)
    assert cv.resident() == {0, 1}
    cv2 = ls.make_buffer("clairvoyant", 2)
    cv2.access(7)
    cv2.access(3)
    cv2.access(5, 10)
    assert cv2.resident() == {3, 5}
    cv2.clear()
    assert cv2.resident() == set() and not cv2.access(3)
    with pytest.raises(ls.ValidationError):
        ls.make_buffer("lru", 0)


def test_optimal_miss_oracle(ls):
    assert ls.optimal_miss_oracle([0, 1, 2, 0, 1], 2) == 3
    assert ls.optimal_miss_oracle([], 2) == 0
    with pytest.raises(ls.CapabilityError):
        ls.optimal_miss_oracle([0] * 17, 2)
    rng = random.Random(77)
    for _ in range(200):
        n, C, k = rng.randint(1, 16), rng.randint(1, 4), rng.randint(1, 6)
        seq = [rng.randrange(k) for _ in range(n)]
        assert ls.optimal_miss_oracle(seq, C) == O.simulate_sequence(seq, C, "clairvoyant"), (seq, C)
