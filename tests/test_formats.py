"""Text artifacts (trace.cpp:72-162, reuse_graph.cpp:103-140, plan.cpp:44-227).

CPU: the readers (lsg_parse_*, host C++ behind the C ABI) on files written by
the UNMODIFIED reference, against the reference's own arrays, and on the
reference's error cases. GPU: the writers (GPU formatters) byte-identical to
the reference's files, and read -> write round trips.
"""
import ctypes
import random

import numpy as np
import pytest

import oracle as O

ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def L():
    import paper_2211_00224_b200 as pkg
    return pkg.lib()


def parse_trace(data: bytes):
    from paper_2211_00224_b200 import _lib
    h = _lib.LsgTraceText()
    rc = L().lsg_parse_trace(data, len(data), ctypes.byref(h), None, 0)
    if rc:
        return rc, L().lsg_last_error().decode(), None
    ids = np.zeros(max(1, h.num_epochs * h.keep), np.uint32)
    assert L().lsg_parse_trace(data, len(data), ctypes.byref(h), ids.ctypes.data_as(ctypes.c_void_p), ids.size) == 0
    return 0, h, ids[: h.num_epochs * h.keep].reshape(h.num_epochs, h.keep)


def parse_plan(data: bytes):
    from paper_2211_00224_b200 import _lib
    h, v = ctypes.c_void_p(), _lib.LsgPlanView()
    rc = L().lsg_parse_plan(data, len(data), ctypes.byref(h), ctypes.byref(v))
    if rc:
        return rc, L().lsg_last_error().decode()
    N, T = v.num_nodes, v.num_steps
    arr = lambda p, n, t: np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(t)), shape=(n,)).copy() if n and p else np.zeros(0, np.dtype(t))  # noqa: E731
    out = dict(items=arr(v.items, v.num_items, ctypes.c_uint32),
               node_off=arr(v.node_off, T * (N + 1), ctypes.c_uint32).reshape(T, N + 1),
               fb=arr(v.fetch_before, T * N, ctypes.c_uint64).reshape(T, N),
               fa=arr(v.fetch_after, T * N, ctypes.c_uint64).reshape(T, N),
               order=arr(v.order, v.num_epochs, ctypes.c_uint32), cost=v.cost, N=N, T=T,
               read_off=arr(v.read_off, T * N + 1, ctypes.c_uint64),
               rs=arr(v.read_start, v.num_reads, ctypes.c_uint64), re=arr(v.read_end, v.num_reads, ctypes.c_uint64),
               needed=arr(v.needed, T * N, ctypes.c_uint64).reshape(T, N),
               redundant=arr(v.redundant, T * N, ctypes.c_uint64).reshape(T, N))
    L().lsg_free_plan(h)
    return 0, out


def rand_cfg(seed):
    r = random.Random(seed)
    N, b = r.choice([1, 2, 3, 4]), r.choice([1, 2, 5, 8])
    B = N * b
    D = B * r.randint(1, 10) + r.randint(0, B - 1)
    return O.Cfg(D, r.randint(1, 5), N, b, seed=r.randint(0, 10**6), buffer_capacity=r.randint(1, max(1, D // 2)),
                 drop_last=r.random() < 0.7, optim_order=r.random() < 0.7, optim_chunk=r.random() < 0.7,
                 chunk_threshold=r.randint(1, 20), pso_iters=20)


@ref
@pytest.mark.parametrize("seed", range(10))
def test_parse_reference_files(seed):
    c = rand_cfg(seed)
    txt, q = O.ref_text(c), O.ref_plan(c)
    rc, h, ids = parse_trace(txt["trace"])
    assert rc == 0 and np.array_equal(ids, q.trace)
    assert (h.dataset_size, h.num_epochs, h.num_nodes, h.local_batch, h.seed, h.drop_last) == (
        c.dataset_size, c.num_epochs, c.num_nodes, c.local_batch, c.seed, int(c.drop_last))
    E = ctypes.c_uint32()
    w = np.zeros(c.num_epochs ** 2, np.uint64)
    assert L().lsg_parse_graph(txt["graph"], len(txt["graph"]), ctypes.byref(E), w.ctypes.data_as(ctypes.c_void_p), w.size) == 0
    assert E.value == c.num_epochs and np.array_equal(w.reshape(E.value, E.value), q.graph)
    rc, p = parse_plan(txt["plan"])
    assert rc == 0
    assert np.array_equal(p["items"], q.items) and np.array_equal(p["node_off"], q.node_off)
    assert np.array_equal(p["fb"], q.fb) and np.array_equal(p["fa"], q.fa)
    assert np.array_equal(p["order"], q.order) and p["cost"] == q.cost
    # reads = the reference's StepPlan.reads (plan_chunks / singles)
    rs, re_, cnt, need, red = O.plan_reads(q.items, q.node_off, c.num_nodes, c.optim_chunk, c.chunk_threshold)
    assert np.array_equal(np.diff(p["read_off"].astype(np.int64)), cnt.ravel())
    assert np.array_equal(p["needed"], need) and np.array_equal(p["redundant"], red)


@pytest.mark.parametrize("text,code,msg", [
    (b"", 3, "missing 'loadsched-trace 1' header"),
    (b"loadsched-trace 2\n", 3, "missing 'loadsched-trace 1' header"),
    (b"loadsched-trace 1\nfoo=1\n", 3, "unknown key 'foo'"),
    (b"loadsched-trace 1\n5\n", 3, "sample id before first epoch header"),
    (b"loadsched-trace 1\ndataset_size=2x\n", 3, "bad integer for dataset_size"),
    (b"loadsched-trace 1\nepoch 1\n", 3, "epoch headers out of order"),
    (b"loadsched-trace 1\nnum_nodes=0\n", 2, "num_nodes must be >= 1"),
    (b"loadsched-trace 1\ndataset_size=4\nnum_epochs=1\nnum_nodes=2\nlocal_batch=2\nepoch 0\n0\n1\n2\n", 3,
     "epoch sequence length mismatch"),
    (b"loadsched-trace 1\ndataset_size=4\nnum_epochs=1\nnum_nodes=2\nlocal_batch=2\nepoch 0\n0\n1\n2\n9\n", 3,
     "sample id out of range"),
    (b"loadsched-trace 1\ndataset_size=4\nnum_epochs=2\nnum_nodes=2\nlocal_batch=2\nepoch 0\n0\n1\n2\n3\n", 3,
     "epoch count does not match"),
])
def test_trace_reader_errors(text, code, msg):
    rc, err, _ = parse_trace(text)
    assert rc == code and msg in err
    if O.ref_available():
        assert O.ref_read("trace", text) == (rc, err)


def test_trace_reader_accepts_reference_grammar():
    # blank lines, a '+' sign and leading blanks are what std::stoull takes
    t = b"loadsched-trace 1\ndataset_size=4\n\nnum_epochs=1\nnum_nodes=2\nlocal_batch= 2\nepoch 0\n+3\n 1\n2\n0\n"
    rc, h, ids = parse_trace(t)
    assert rc == 0 and ids.tolist() == [[3, 1, 2, 0]] and h.drop_last == 1


HEAD = b"loadsched-plan 1\nmeta dataset_size=8 nodes=2 local_batch=2 threshold=4\norder: 0\ncost: 0\n"


@pytest.mark.parametrize("body,msg", [
    (b"", "order length != epoch count"),
    (b"assign 0 0 0 1 hit\n", None),
    (b"assign 0 0 2 1 hit\n", "assign row node out of range"),
    (b"assign 0 0 0 1 maybe\n", "bad source tag: maybe"),
    (b"assign 0 0 0 1x hit\n", "bad source tag: x"),
    (b"assign 0 0 0\n", "bad assign row"),
    (b"balance 0 0 0 1\n", "bad balance row"),
    (b"read 0 0 0 chunk 5 3\n", "read row end < start"),
    (b"read 0 0 0 big 1 3\n", "bad read kind: big"),
    (b"assign 0 0 0 1 fetch\nassign 0 0 0 1 fetch\nread 0 0 0 chunk 1 1\n", "read rows inconsistent with fetches"),
    (b"assign 0 0 0 3 fetch\nread 0 0 0 chunk 1 2\n", None),
    (b"assign 1 0 0 3 fetch\n", "epoch rows out of schedule order"),
    (b"assign 0 0 0 3 fetch\nassign 1 0 0 2 fetch\n", "order length != epoch count"),
    (b"frob 1\n", "unknown row tag: frob"),
    (b"   \n", "unknown row tag: "),
])
def test_plan_reader_errors(body, msg):
    r = parse_plan(HEAD + body)
    if msg is None:
        assert r[0] == 0
    else:
        assert r[0] == 3 and msg in r[1], r
    if O.ref_available():  # the reference reader agrees, message included
        code, rmsg = O.ref_read("plan", HEAD + body)
        assert code == r[0] and (msg is None or rmsg == r[1]), (code, rmsg, r)


def test_plan_reader_header_errors():
    assert parse_plan(b"loadsched-plan 2\n")[0] == 3
    r = parse_plan(b"loadsched-plan 1\nassign 0 0 0 1 hit\n")
    assert r[0] == 3 and "assign row before meta" in r[1]
    r = parse_plan(b"loadsched-plan 1\nmeta dataset_size=8 nodes=0\n")
    assert r[0] == 3 and "meta missing nodes" in r[1]
    r = parse_plan(b"loadsched-plan 1\nmeta dataset_size=8 nodes=1 color=3\n")
    assert r[0] == 3 and "unknown meta key: color" in r[1]
    r = parse_plan(b"loadsched-plan 1\nmeta nodes=1\norder: 0\n")
    assert r[0] == 3 and "missing meta/order/cost" in r[1]
    r = parse_plan(HEAD.replace(b"order: 0", b"order: 1 0") + b"assign 0 0 0 1 hit\nassign 1 0 0 2 hit\n")
    assert r[0] == 3 and "epoch rows out of schedule order" in r[1]


# ------------------------------------------------------------- GPU writers --
@ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(10))
def test_writers_match_reference_files(ls, seed):
    from test_gpu_parity import to_pc
    c = rand_cfg(seed)
    out = ls.plan_schedule(to_pc(ls, c))
    txt = O.ref_text(c)
    assert ls.format_trace(out.trace) == txt["trace"]
    assert ls.format_graph(out.graph) == txt["graph"]
    assert ls.format_plan(out.plan) == txt["plan"]
    # run reports: metrics.csv of the configured pass and the cost totals
    pol = c.policy
    sim = ls.simulate_plan(out.plan, c.buffer_capacity, pol,
                           insert_redundant=bool(c.chunk_insert_redundant and c.optim_chunk))
    assert ls.format_metrics(out.plan, sim, pol) == txt["metrics"]
    costs = b"%.6f %.6f\n" % (ls.total_barrier_cost(out.plan), ls.total_io_cost(out.plan))
    assert costs == txt["costs"]


@ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed,policy,red", [(1, "lru", False), (2, "clairvoyant", True), (3, "lru", False),
                                             (4, "clairvoyant", True)])
def test_metrics_match_reference(ls, seed, policy, red):
    """write_metrics (pipeline.cpp:153-179) and total_barrier_cost /
    total_io_cost of LRU and redundant-insert passes, byte for byte."""
    import dataclasses
    from test_gpu_parity import to_pc
    c = dataclasses.replace(rand_cfg(seed), policy=policy, chunk_insert_redundant=red, optim_chunk=True)
    out = ls.plan_schedule(to_pc(ls, c))
    txt = O.ref_text(c)
    sim = ls.simulate_plan(out.plan, c.buffer_capacity, policy, insert_redundant=red)
    assert ls.format_metrics(out.plan, sim, policy) == txt["metrics"]
    assert b"%.6f %.6f\n" % (ls.total_barrier_cost(out.plan), ls.total_io_cost(out.plan)) == txt["costs"]
    assert ls.format_metrics(out.plan, sim, policy, ls.CostModel(2.5, 0.125)).count(b"\n") == \
        1 + out.plan.node_off.shape[0] * out.plan.num_nodes


@ref
@pytest.mark.gpu
@pytest.mark.parametrize("seed,seek,stream", [(5, 0.37, 0.0013), (6, 13.0, 1.0), (7, 1e-3, 7.25)])
def test_cost_totals_bit_exact(ls, seed, seek, stream):
    """total_barrier_cost / total_io_cost (pipeline.cpp:133-151) summed on the
    device (lsg_plan_costs) equal the reference's doubles bit for bit under a
    non-integer cost model (no FMA contraction, reference summation order)."""
    from test_gpu_parity import to_pc
    c = rand_cfg(seed)
    out = ls.plan_schedule(to_pc(ls, c))
    txt = O.ref_text(c, (f"seek_cost={seek!r}", f"stream_cost={stream!r}"))
    m = ls.CostModel(seek, stream)
    got = ("%s %s\n" % (float.hex(ls.total_barrier_cost(out.plan, m)), float.hex(ls.total_io_cost(out.plan, m))))
    want = txt["costs_exact"].decode()
    assert [float.fromhex(x) for x in got.split()] == [float.fromhex(x) for x in want.split()], (got, want)


@pytest.mark.gpu
def test_plan_file_round_trip_and_replay(ls, tmp_path):
    """read_plan(write_plan(p)) replays to the same SimResult rows; the
    cfg2-shaped plan file (E=4) is formatted on the GPU."""
    from test_gpu_parity import u32
    pc = ls.PipelineConfig(trace=ls.TraceConfig(262144, 4, 8, 512, 42, True), buffer_capacity=52428)
    out = ls.plan_schedule(pc)
    path = tmp_path / "plan.txt"
    ls.write_plan_file(path, out.plan)
    back = ls.read_plan_file(path)
    assert np.array_equal(u32(back.items), u32(out.plan.items))
    assert np.array_equal(u32(back.node_off), u32(out.plan.node_off))
    a = ls.simulate_plan(out.plan, 52428)
    b = ls.simulate_plan(back, 52428)
    assert np.array_equal(u32(a.hits), u32(b.hits)) and np.array_equal(u32(a.misses), u32(b.misses))
    assert ls.format_plan(back) == path.read_bytes()
    t = tmp_path / "trace.txt"
    ls.write_trace_file(t, out.trace)
    assert np.array_equal(u32(ls.read_trace_file(t).epochs), u32(out.trace.epochs))
