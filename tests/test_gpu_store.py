"""The Store (store.hpp:13-81) on the B200 path: create_store byte-identical
to the reference's file, open/read_one/read_chunk semantics and error
classes (tests/test_store.cpp), reads of sample sets straight into HBM, and
the step fetch with its misses read from the file — every batch row equal to
Store::read_one of its id."""
import os
import random

import numpy as np
import pytest

import oracle as O
from test_gpu_parity import to_pc, u32

pytestmark = pytest.mark.gpu


@pytest.fixture
def tmp(tmp_path):
    return str(tmp_path)


@pytest.mark.parametrize("count,size,seed", [(1, 1, 0), (5, 24, 77), (16, 7, 1), (1000, 256, 3),
                                             (3, (64 << 20) // 3 + 5, 9)])
def test_create_store_matches_reference_file(ls, tmp, count, size, seed):
    mine, ref = os.path.join(tmp, "mine.bin"), os.path.join(tmp, "ref.bin")
    ls.create_store(mine, count, size, seed, max_bytes=1 << 40)
    if O.ref_available():
        O.ref_store_file(ref, count, size, seed)
        assert open(mine, "rb").read() == open(ref, "rb").read()
    raw = open(mine, "rb").read()
    assert raw[:4] == b"SLRD" and raw[4:6] == b"\x01\x00"
    assert int.from_bytes(raw[6:14], "little") == count and int.from_bytes(raw[14:22], "little") == size
    want = O.store_payload(seed, 0, count * size)
    assert np.array_equal(np.frombuffer(raw[22:], np.uint8), want)


def test_store_golden_and_reads(ls, tmp):
    """tests/test_store.cpp:63-65 golden payload, :73-91 chunk == singles."""
    p = os.path.join(tmp, "s.bin")
    ls.create_store(p, 8, 16, 1)
    with ls.Store(p) as s:
        assert s.sample_count == 8 and s.sample_size == 16 and s.header().version == 1
        first = s.read_one(0) + s.read_one(1)
        assert first.hex() == "c15c0289ec2d0a9167ec8e65a18debbe5e5532fbeea293f80bc942ee9086c171"
        assert s.read_chunk(2, 5) == b"".join(s.read_one(i) for i in range(2, 7))
        with pytest.raises(ls.ValidationError):
            s.read_one(8)
        with pytest.raises(ls.ValidationError):
            s.read_chunk(6, 3)
        with pytest.raises(ls.ValidationError):
            s.read_chunk(0, 0)


def test_store_errors(ls, tmp):
    with pytest.raises(ls.StorageError):
        ls.create_store(os.path.join(tmp, "a"), 0, 4, 1)
    with pytest.raises(ls.StorageError):
        ls.create_store(os.path.join(tmp, "b"), 1 << 20, 1 << 20, 1)  # over the 1 GiB budget
    with pytest.raises(ls.StorageError):
        ls.Store(os.path.join(tmp, "missing"))
    p = os.path.join(tmp, "bad")
    ls.create_store(p, 4, 8, 1)
    raw = bytearray(open(p, "rb").read())
    open(p + "m", "wb").write(b"XLRD" + raw[4:])
    with pytest.raises(ls.StorageError):
        ls.Store(p + "m")
    open(p + "v", "wb").write(raw[:4] + b"\x02\x00" + raw[6:])
    with pytest.raises(ls.StorageError):
        ls.Store(p + "v")
    open(p + "t", "wb").write(raw[:-1])
    with pytest.raises(ls.StorageError):
        ls.Store(p + "t")


@pytest.mark.parametrize("thr", [1, 4, 15, 1000])
def test_read_rows_into_hbm(ls, tmp, thr):
    p = os.path.join(tmp, "r.bin")
    count, size = 5000, 48
    ls.create_store(p, count, size, 5)
    payload = O.store_payload(5, 0, count * size).reshape(count, size)
    r = np.random.default_rng(thr)
    ids = r.integers(0, count, size=700).astype(np.uint32)  # repeats, any order
    with ls.Store(p) as s:
        got = s.read_rows(ids, threshold=thr).cpu().numpy()
        assert np.array_equal(got, payload[ids])
        with pytest.raises(ls.ValidationError):
            s.read_rows(np.array([count], np.uint32))


@pytest.mark.parametrize("seed", range(3))
def test_fetch_steps_with_misses_from_the_store(ls, tmp, seed):
    """Whole plans: every step's batch rows (hits from the HBM buffer, misses
    from the Store file) equal Store::read_one of the row's id."""
    import torch
    r = random.Random(seed)
    N, b = r.choice([2, 4]), r.choice([8, 16])
    D = N * b * r.randint(4, 10)
    C = r.randint(N * b, D // 2)
    SB = 64
    c = O.Cfg(D, 3, N, b, seed=seed, buffer_capacity=C, pso_iters=10)
    out = ls.plan_schedule(to_pc(ls, c))
    sim = ls.simulate_plan(out.plan, C, want_slots=True)
    p = os.path.join(tmp, "f.bin")
    ls.create_store(p, D, SB, 11)
    payload = O.store_payload(11, 0, D * SB).reshape(D, SB)
    bufs = [torch.zeros((C, SB), dtype=torch.uint8, device="cuda") for _ in range(N)]
    outs = [torch.zeros((4 * b, SB), dtype=torch.uint8, device="cuda") for _ in range(N)]
    off = u32(out.plan.node_off)
    items = u32(out.plan.items) & 0x7FFFFFFF
    with ls.Store(p) as s:
        fetch = ls.StepFetcher(bufs, outs, (0, N), SB, 11, store=s, threshold=5)
        base = 0
        for g in range(off.shape[0]):
            fetch(out.plan.items[base:], sim.slots[base:], out.plan.node_off[g], int(off[g, N]))
            for k in range(N):
                n = int(off[g, k + 1] - off[g, k])
                ids = items[base + off[g, k]: base + off[g, k + 1]]
                assert np.array_equal(outs[k][:n].cpu().numpy(), payload[ids]), (g, k)
            base += int(off[g, N])
