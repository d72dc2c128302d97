"""GPU parity for K7 (per-rank replay), K9 (store payload) and K8 (gather),
and the end-to-end HBM buffer data path (replay slots + fill + gather)."""
import random

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import to_pc, u32

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).cuda()


def _plan_obj(ls, items, node_off, N, D, spe):
    T = node_off.shape[0]
    return ls.SchedulePlan(D, N, 0, spe, None, _dev(items), _dev(node_off.reshape(T, N + 1)), None, None)


@pytest.mark.parametrize("seed", range(30))
def test_replay_matches_oracle_on_oracle_plans(ls, seed):
    r = random.Random(77 + seed)
    N, b = r.choice([1, 2, 3, 4, 8]), r.choice([1, 2, 4, 8, 16])
    B = N * b
    D = B * r.randint(1, 25) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 7), N, b, seed=seed, buffer_capacity=r.randint(1, max(1, D // 3)),
              drop_last=r.random() < 0.7, optim_order=r.random() < 0.7,
              optim_remap=r.random() < 0.8, optim_balance=r.random() < 0.8, pso_iters=20)
    p = O.plan(c)
    for C in (c.buffer_capacity, max(1, c.buffer_capacity // 3), D):
        h, m = O.simulate(p.items, p.node_off, N, D, C)
        sim = ls.simulate_plan(_plan_obj(ls, p.items, p.node_off, N, D, c.steps), C)
        assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m), C


def test_replay_readme_demo_totals(ls):
    c = O.Cfg(1024, 6, 4, 8, seed=7, buffer_capacity=64)
    out = ls.plan_schedule(to_pc(ls, c))
    sim = ls.simulate_plan(out.plan, 64)
    assert (sim.total_misses, sim.total_hits) == (4864, 1280)


def test_replay_whole_dataset_buffer_only_cold_misses(ls):
    # tests/test_pipeline.cpp:164-173
    c = O.Cfg(64, 3, 1, 8, seed=5, buffer_capacity=64)
    out = ls.plan_schedule(to_pc(ls, c))
    sim = ls.simulate_plan(out.plan, 64)
    assert sim.total_misses == 64 and sim.total_hits == 3 * 64 - 64


def test_replay_node_range_sharding(ls):
    c = O.Cfg(4096, 5, 8, 16, seed=11, buffer_capacity=300)
    out = ls.plan_schedule(to_pc(ls, c))
    full = ls.simulate_plan(out.plan, 300)
    parts = [ls.simulate_plan(out.plan, 300, node_range=(k0, k1)) for k0, k1 in ((0, 3), (3, 8))]
    hits = u32(parts[0].hits).copy()
    hits[:, 3:] = u32(parts[1].hits)[:, 3:]
    assert np.array_equal(hits, u32(full.hits))


def test_replay_rejects_repeats_within_a_step(ls):
    items = np.array([1, 1, 2, 3], dtype=np.uint32)
    off = np.array([[0, 2, 4]], dtype=np.uint32)
    with pytest.raises(ls.Error):
        ls.simulate_plan(_plan_obj(ls, items, off, 2, 8, 1), 2)


def test_store_fill_golden(ls):
    import torch
    # tests/test_store.cpp:63-65 — first 32 payload bytes of a seed-1 store
    row = ls.store_fill(torch.tensor([0], dtype=torch.int32, device="cuda"), 32, 1)
    assert bytes(row.cpu().numpy().ravel()).hex() == \
        "c15c0289ec2d0a9167ec8e65a18debbe5e5532fbeea293f80bc942ee9086c171"


@pytest.mark.parametrize("size", [16, 48, 4096, 7, 1000])
def test_store_fill_matches_oracle(ls, size):
    import torch
    ids = np.array([5, 0, 17, 3, 17, 99], dtype=np.uint32)
    got = ls.store_fill(_dev(ids), size, 12345).cpu().numpy()
    for r, x in enumerate(ids):
        assert np.array_equal(got[r], O.store_payload(12345, int(x) * size, size))


def test_gather_matches_indexing(ls):
    import torch
    g = torch.Generator(device="cuda").manual_seed(0)
    buf = torch.randint(0, 255, (257, 262144), dtype=torch.uint8, device="cuda", generator=g)
    slots = torch.randint(0, 257, (300,), dtype=torch.int32, device="cuda", generator=g)
    out = ls.gather(buf, slots, 262144)
    assert torch.equal(out, buf[slots.long()])
    small = torch.randint(0, 255, (10, 48), dtype=torch.uint8, device="cuda", generator=g)
    s2 = torch.tensor([9, 0, 3, 3], dtype=torch.int32, device="cuda")
    assert torch.equal(ls.gather(small, s2, 48), small[s2.long()])


@pytest.mark.parametrize("seed", range(4))
def test_buffer_data_path_end_to_end(ls, seed):
    """Replay slots drive a real per-node HBM buffer: every step, the samples
    resident at step start are gathered from their slots (bytes must equal
    Store::read_one), then misses are 'fetched' (K9) into their new slots."""
    import torch
    r = random.Random(seed)
    N, b = r.choice([2, 4]), r.choice([4, 8])
    D = N * b * r.randint(4, 10)
    C = r.randint(N * b, D // 2)
    size, fill_seed, NEV = 64, 99, 0xFFFFFFFE
    c = O.Cfg(D, 4, N, b, seed=seed, buffer_capacity=C, pso_iters=20)
    out = ls.plan_schedule(to_pc(ls, c))
    sim = ls.simulate_plan(out.plan, C, want_slots=True)
    items = u32(out.plan.items) & 0x7FFFFFFF
    slots = u32(sim.slots)
    off = u32(out.plan.node_off)
    hits = u32(sim.hits)
    bufs = [torch.zeros((C, size), dtype=torch.uint8, device="cuda") for _ in range(N)]
    owner = [dict() for _ in range(N)]
    base = 0
    for g in range(off.shape[0]):
        for k in range(N):
            lo, hi = base + off[g, k], base + off[g, k + 1]
            ids, raw = items[lo:hi], slots[lo:hi]
            hitf = (raw != NEV) & ((raw >> 31) == 1)
            sl = np.where(raw == NEV, NEV, raw & 0x7FFFFFFF)
            assert all(s == NEV or s < C for s in sl)
            want = ls.store_fill(_dev(ids), size, fill_seed)
            res = [i for i in range(len(ids)) if hitf[i]]
            assert len(res) == hits[g, k], (g, k)
            assert all(owner[k].get(int(sl[i])) == int(ids[i]) for i in res), (g, k)
            if res:
                got = ls.gather(bufs[k], _dev(sl[res]), size)
                assert torch.equal(got, want[res]), (g, k)
            miss = [i for i in range(len(ids)) if i not in set(res) and sl[i] != NEV]
            if miss:
                bufs[k][torch.from_numpy(sl[miss].astype(np.int64)).cuda()] = want[miss]
                for i in miss:
                    owner[k][int(sl[i])] = int(ids[i])
        base += off[g, N]


@pytest.mark.parametrize("seed,rng", [(0, None), (1, (1, 3)), (2, None)])
def test_fetch_step_end_to_end(ls, seed, rng):
    """lsg_fetch_step over the whole job: after every step each local rank's
    batch rows equal Store::read_one of its list (hits from HBM slots, misses
    from storage), i.e. the HBM buffers stay consistent with the replay."""
    import torch
    r = random.Random(100 + seed)
    N, b = 4, r.choice([4, 8])
    D = N * b * r.randint(5, 9)
    C = r.randint(N * b, D // 2)
    SB, fill = 48, 5
    c = O.Cfg(D, 5, N, b, seed=seed, buffer_capacity=C, pso_iters=20)
    out = ls.plan_schedule(to_pc(ls, c))
    k0, k1 = rng or (0, N)
    sim = ls.simulate_plan(out.plan, C, node_range=(k0, k1), want_slots=True)
    bufs = [torch.zeros((C, SB), dtype=torch.uint8, device="cuda") for _ in range(k0, k1)]
    outs = [torch.zeros((N * b, SB), dtype=torch.uint8, device="cuda") for _ in range(k0, k1)]
    fetch = ls.StepFetcher(bufs, outs, (k0, k1), SB, fill)
    off = u32(out.plan.node_off)
    items = u32(out.plan.items) & 0x7FFFFFFF
    base = 0
    for g in range(off.shape[0]):
        fetch(out.plan.items[base:], sim.slots[base:], out.plan.node_off[g], int(off[g, k1] - off[g, k0]))
        for k in range(k0, k1):
            lo, hi = base + off[g, k], base + off[g, k + 1]
            want = ls.store_fill(_dev(items[lo:hi]), SB, fill)
            assert torch.equal(outs[k - k0][: hi - lo], want), (g, k)
        base += off[g, N]


@pytest.mark.parametrize("SB", [48, 8192 * 2])
def test_fetch_steps_matches_per_step(ls, SB):
    """lsg_fetch_steps (one C call over a step range) leaves the HBM buffers
    exactly as the per-step lsg_fetch_step loop does, the last step's batch
    rows too, and those equal Store::read_one of its lists. (Rows past the
    last step's list are unspecified: over a range, steps alternate between
    the batch tensors and a scratch set, the last one landing in the
    tensors.)"""
    import torch
    N, b, D, C, fill = 4, 8, 4 * 8 * 7, 60, 9
    c = O.Cfg(D, 4, N, b, seed=3, buffer_capacity=C, pso_iters=20)
    out = ls.plan_schedule(to_pc(ls, c))
    k0, k1 = 1, 4
    sim = ls.simulate_plan(out.plan, C, node_range=(k0, k1), want_slots=True)
    off = u32(out.plan.node_off)
    T = off.shape[0]
    res = []
    for mode in ("step", "range"):
        bufs = [torch.zeros((C, SB), dtype=torch.uint8, device="cuda") for _ in range(k0, k1)]
        outs = [torch.zeros((N * b, SB), dtype=torch.uint8, device="cuda") for _ in range(k0, k1)]
        f = ls.StepFetcher(bufs, outs, (k0, k1), SB, fill)
        if mode == "step":
            base = 0
            for g in range(T):
                f(out.plan.items[base:], sim.slots[base:], out.plan.node_off[g], int(off[g, k1] - off[g, k0]))
                base += off[g, N]
        else:
            f.fetch_steps(out.plan, sim.slots, off, 0, T // 2)
            f.fetch_steps(out.plan, sim.slots, off, T // 2, T)
        torch.cuda.synchronize()
        res.append((bufs, outs))
    for a, z in zip(res[0][0], res[1][0]):
        assert torch.equal(a, z)
    for k in range(k0, k1):
        n = int(off[T - 1, k + 1] - off[T - 1, k])
        assert torch.equal(res[0][1][k - k0][:n], res[1][1][k - k0][:n])
    items = u32(out.plan.items) & 0x7FFFFFFF
    base = int(off[:-1, N].sum())
    for k in range(k0, k1):
        lo, hi = base + off[T - 1, k], base + off[T - 1, k + 1]
        want = ls.store_fill(_dev(items[lo:hi]), SB, fill)
        assert torch.equal(res[1][1][k - k0][: hi - lo], want)
    with pytest.raises(ls.ValidationError):
        f.fetch_steps(out.plan, sim.slots, off, 3, 2)


@pytest.mark.parametrize("variant", ["chain", "tables"])
@pytest.mark.parametrize("seed", range(12))
def test_cta_replay_variants(ls, monkeypatch, variant, seed):
    """The per-rank CTA replay in both forms — the chain replay (residency
    from the key-space bitmap, slots written ahead; the default for long
    lists) and round 1's id-indexed tables — forced onto short-list plans:
    hits/misses equal the oracle's and the slots drive a consistent HBM
    buffer (every hit's slot holds its sample)."""
    monkeypatch.setenv("LSG_REPLAY_CTA", "1")
    if variant == "tables":
        monkeypatch.setenv("LSG_REPLAY_TABLES", "1")
    r = random.Random(500 + seed)
    N, b = r.choice([1, 2, 3, 4, 8]), r.choice([1, 2, 4, 8, 16])
    B = N * b
    D = B * r.randint(2, 25) + r.randint(0, B - 1)
    c = O.Cfg(D, r.randint(1, 7), N, b, seed=seed, buffer_capacity=r.randint(1, max(1, D // 3)),
              drop_last=r.random() < 0.7, optim_order=r.random() < 0.7,
              optim_remap=r.random() < 0.8, optim_balance=r.random() < 0.8, pso_iters=20)
    p = O.plan(c)
    for C in (c.buffer_capacity, max(1, c.buffer_capacity // 3), D):
        h, m = O.simulate(p.items, p.node_off, N, D, C)
        sim = ls.simulate_plan(_plan_obj(ls, p.items, p.node_off, N, D, c.steps), C, want_slots=True)
        assert np.array_equal(u32(sim.hits), h) and np.array_equal(u32(sim.misses), m), C
        slots = u32(sim.slots)
        owner = [dict() for _ in range(N)]
        base = 0
        for g in range(p.node_off.shape[0]):
            for k in range(N):
                lo, hi = base + p.node_off[g, k], base + p.node_off[g, k + 1]
                ids = p.items[lo:hi] & 0x7FFFFFFF
                raw = slots[lo:hi]
                hit = (raw != 0xFFFFFFFE) & ((raw >> 31) == 1)
                for i in range(len(ids)):
                    if hit[i]:
                        assert owner[k].get(int(raw[i] & 0x7FFFFFFF)) == int(ids[i]), (C, g, k, i)
                for i in range(len(ids)):
                    if not hit[i] and raw[i] != 0xFFFFFFFE:
                        assert raw[i] < C
                        owner[k][int(raw[i])] = int(ids[i])
            base += p.node_off[g, N]
