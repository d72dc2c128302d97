"""GPU byte checks of the batch fetch (the reference's Store::read_one /
read_chunk bytes, store.cpp:123-148, payload store.cpp:70-80) through the
whole-job path (lsg_fetch_job / lsg_fetch_steps):

* at the BENCH shape — 256 KiB rows (so the TMA bulk-copy hit kernel runs,
  32 tiles per row, guided chunk claims over 296 CTAs), 8 ranks, local batch
  256, 56 consecutive steps — every batch row of every rank after every step
  equals the Store payload of its sample id;
* with the HOST TIER as the miss source (the dataset's payload rows in a
  pinned tmpfs file, read over PCIe by the TMA prefetcher into a ring),
  including a ring far smaller than the job (wrap-around) and rows that are
  not whole TMA tiles (the LSU prefetcher), and the final buffer contents;
* the job statistics (misses, kept misses, host bytes, hits) against the
  replay's counts.
"""
import os
import tempfile

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu


def u32(t):
    return t.detach().cpu().numpy().view(np.uint32)


def setup(ls, D, E, N, b, frac, seed=42):
    pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, seed, True), buffer_capacity=int(frac * D))
    out = ls.plan_schedule(pc)
    sim = ls.simulate_plan(out.plan, pc.buffer_capacity, want_slots=True)
    return pc, out.plan, sim


def tensors(N, C, maxlen, SB, dev="cuda"):
    bufs = [torch.zeros((C, SB), dtype=torch.uint8, device=dev) for _ in range(N)]
    outs = [torch.zeros((maxlen, SB), dtype=torch.uint8, device=dev) for _ in range(N)]
    return bufs, outs


def check_step(ls, plan, off, g, outs, k0, k1, SB, fill_seed=1):
    """Rows of step g of ranks [k0, k1) == Store payload of their ids."""
    base = int(off[:g, -1].astype(np.int64).sum())
    ids = plan.items[base:base + int(off[g, -1])] & 0x7FFFFFFF
    for k in range(k0, k1):
        lo, hi = int(off[g, k]), int(off[g, k + 1])
        if hi == lo:
            continue
        want = ls.store_fill(ids[lo:hi], SB, fill_seed)
        got = outs[k - k0][: hi - lo]
        if not torch.equal(got, want):
            bad = (got != want).any(dim=1).nonzero().flatten().tolist()
            raise AssertionError(f"step {g} rank {k}: rows {bad[:8]} differ from Store::read_one")


def test_bench_shape_tma_fetch_every_step(ls):
    """256 KiB rows, 8 ranks, b = 256: 56 steps, every row of every rank."""
    D, E, N, b, SB = 16384, 7, 8, 256, 256 * 1024
    pc, plan, sim = setup(ls, D, E, N, b, 0.20)
    off = u32(plan.node_off)
    T = off.shape[0]
    assert T == 56
    assert int((off[:, 1:] - off[:, :-1]).max()) <= 2 * b
    bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, SB)
    f = ls.StepFetcher(bufs, outs, (0, N), SB, 1)
    hits = misses = 0
    for g in range(T):
        f.fetch_steps(plan, sim.slots, off, g, g + 1)  # lsg_fetch_steps: the bench's path
        check_step(ls, plan, off, g, outs, 0, N, SB)
    torch.cuda.synchronize()
    hits, misses = sim.total_hits, sim.total_misses
    assert hits > 10 * 2 * b and misses > 0  # the TMA hit kernel did real work


def test_whole_job_final_buffers(ls):
    """One lsg_fetch_steps call over the whole job: the last step's batch and
    every buffer slot's final content (the last sample written to it)."""
    D, E, N, b, SB = 4096, 6, 4, 64, 8192
    pc, plan, sim = setup(ls, D, E, N, b, 0.1)
    off = u32(plan.node_off)
    T = off.shape[0]
    bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, SB)
    ls.StepFetcher(bufs, outs, (0, N), SB, 1).fetch_steps(plan, sim.slots, off)
    check_step(ls, plan, off, T - 1, outs, 0, N, SB)
    check_final_slots(ls, plan, sim, off, bufs, 0, N, SB)


def check_final_slots(ls, plan, sim, off, bufs, k0, k1, SB, fill_seed=1):
    items = u32(plan.items) & 0x7FFFFFFF
    slots = u32(sim.slots)
    T, N = off.shape[0], off.shape[1] - 1
    bases = np.concatenate([[0], np.cumsum(off[:, N].astype(np.int64))])
    for k in range(k0, k1):
        last = {}
        for g in range(T):
            lo, hi = bases[g] + off[g, k], bases[g] + off[g, k + 1]
            for sl, x in zip(slots[lo:hi].tolist(), items[lo:hi].tolist()):
                if sl != 0xFFFFFFFE and not sl >> 31:
                    last[sl] = x
        if not last:
            continue
        s = torch.tensor(sorted(last), dtype=torch.int64, device="cuda")
        want = ls.store_fill(torch.tensor([last[i] for i in sorted(last)], dtype=torch.int32, device="cuda"), SB,
                             fill_seed)
        assert torch.equal(bufs[k - k0][s], want), f"rank {k}: final slot contents"


@pytest.fixture
def host_rows(ls):
    made = []

    def make(D, SB):
        d = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        path = os.path.join(d, f"lsg_test_rows_{os.getpid()}_{len(made)}")
        h = ls.HostRows(path, D, SB, 1, create=True)
        made.append(h)
        return h
    yield make
    for h in made:
        h.close()
        os.remove(h.path)


def test_host_rows_bytes_are_the_store_payload(ls, host_rows):
    h = host_rows(300, 4096)
    v = h.view()
    assert np.array_equal(v[7], O.store_payload(1, 7 * 4096, 4096))
    assert np.array_equal(v[299], O.store_payload(1, 299 * 4096, 4096))
    with pytest.raises(ls.StorageError):
        ls.HostRows(h.path, 301, 4096, 1, create=False)  # wrong length


@pytest.mark.parametrize("SB,ring", [(8192, 0), (8192, 8192 * 48), (1024, 1024 * 40), (256 * 1024, 0)])
def test_host_tier_misses_every_step(ls, host_rows, SB, ring):
    """Misses read from the pinned host rows by the prefetcher (TMA for 8 KiB
    multiples, LSU otherwise), ring wrap-around included: one job per step,
    every batch row checked; then one whole-job call and the final slots."""
    D, E, N, b = 2048, 5, 4, 32
    pc, plan, sim = setup(ls, D, E, N, b, 0.15)
    off = u32(plan.node_off)
    T = off.shape[0]
    h = host_rows(D, SB)
    bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, SB)
    k0, k1 = 1, 4  # a node range, as one GPU of several would own
    bl, ol = bufs[k0:k1], outs[k0:k1]
    tot = {"misses": 0, "kept": 0, "host_bytes": 0, "hits": 0}
    for g in range(T):
        j = ls.FetchJob(bl, ol, (k0, k1), plan, sim.slots, off, SB, 1, host=h, step_range=(g, g + 1),
                        ring_bytes=ring)
        j.run()
        for key, v in j.stats().items():
            tot[key] += v
        j.close()
        check_step(ls, plan, off, g, ol, k0, k1, SB)
    hits = u32(sim.hits)[:, k0:k1].sum()
    misses = u32(sim.misses)[:, k0:k1].sum()
    assert tot["hits"] == hits and tot["misses"] == misses and tot["host_bytes"] == misses * SB
    # the whole job in one call (ring far smaller than the job when ring > 0)
    for t in bufs + outs:
        t.zero_()
    prep = torch.cuda.Stream()
    j = ls.FetchJob(bl, ol, (k0, k1), plan, sim.slots, off, SB, 1, host=h, prep_stream=prep, ring_bytes=ring)
    j.run()
    st = j.stats()
    j.close()
    torch.cuda.synchronize()
    assert st["misses"] == misses
    check_step(ls, plan, off, T - 1, ol, k0, k1, SB)
    check_final_slots(ls, plan, sim, off, bl, k0, k1, SB)


def test_host_tier_wrong_sample_size(ls, host_rows):
    D, E, N, b = 512, 2, 2, 16
    pc, plan, sim = setup(ls, D, E, N, b, 0.2)
    h = host_rows(D, 4096)
    bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, 8192)
    with pytest.raises(ls.ValidationError):
        ls.FetchJob(bufs, outs, (0, N), plan, sim.slots, u32(plan.node_off), 8192, 1, host=h)


@pytest.mark.parametrize("SB,ring_rows", [(8192, 96), (1024, 70)])
def test_shared_miss_stream_across_jobs(ls, host_rows, SB, ring_rows):
    """Consecutive jobs through one MissStream (ring far smaller than a job,
    sequence numbers running on across jobs, every job created before the
    previous one has fetched): each job's last batch and final buffer
    contents are the Store payload."""
    D, E, N, b = 2048, 4, 2, 32
    h = host_rows(D, SB)
    ms = ls.MissStream(SB, ring_rows * SB)
    fstream = torch.cuda.current_stream()
    jobs = []
    for seed in (1, 2, 3):
        pc, plan, sim = setup(ls, D, E, N, b, 0.2, seed=seed)
        off = u32(plan.node_off)
        bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, SB)
        prep = torch.cuda.Stream()
        j = ls.FetchJob(bufs, outs, (0, N), plan, sim.slots, off, SB, 1, host=h, prep_stream=prep, misses=ms)
        jobs.append((j, plan, sim, off, bufs, outs))
    for j, *_ in jobs:
        j.run()
    torch.cuda.synchronize()
    for j, plan, sim, off, bufs, outs in jobs:
        assert j.stats()["misses"] == int(u32(sim.misses).sum())
        j.close()
        check_step(ls, plan, off, off.shape[0] - 1, outs, 0, N, SB)
        check_final_slots(ls, plan, sim, off, bufs, 0, N, SB)
    ms.close()


def test_large_rows_synthesised_misses(ls):
    """Rows above 1 MiB with synthesised misses (the cfg3 shape in small):
    the producer warps compute 2 MiB payload rows tile by tile beside the hit
    copies; every step's batch and the final slots are the Store payload."""
    D, E, N, b, SB = 512, 4, 2, 8, 2 << 20
    pc, plan, sim = setup(ls, D, E, N, b, 0.2)
    off = u32(plan.node_off)
    T = off.shape[0]
    bufs, outs = tensors(N, pc.buffer_capacity, 2 * b, SB)
    f = ls.StepFetcher(bufs, outs, (0, N), SB, 1)
    for g in range(0, T, 5):
        f.fetch_steps(plan, sim.slots, off, g, min(T, g + 5))
        check_step(ls, plan, off, min(T, g + 5) - 1, outs, 0, N, SB)
    check_final_slots(ls, plan, sim, off, bufs, 0, N, SB)
