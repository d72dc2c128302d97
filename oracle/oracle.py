"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the C restatement (oracle/liboracle.so, the "port") and a
subprocess wrapper around the compiled reference driver (oracle/_ref/ref_dump,
the "reference"). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs may import this module; the product package
never does.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
import tempfile
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_DUMP = os.path.join(HERE, "_ref", "ref_dump")
HIT_BIT = 0x80000000
NEVER = 0xFFFFFFFFFFFFFFFF


class OrConfig(ctypes.Structure):
    """Field-for-field mirror of or_config (solar_oracle.h)."""

    _fields_ = [
        ("dataset_size", ctypes.c_uint64),
        ("num_epochs", ctypes.c_uint32),
        ("num_nodes", ctypes.c_uint32),
        ("local_batch", ctypes.c_uint64),
        ("seed", ctypes.c_uint64),
        ("drop_last", ctypes.c_int32),
        ("policy", ctypes.c_int32),
        ("buffer_capacity", ctypes.c_uint64),
        ("graph_mode", ctypes.c_int32),
        ("insert_redundant", ctypes.c_int32),
        ("chunk_threshold", ctypes.c_uint64),
        ("optim_order", ctypes.c_int32),
        ("optim_remap", ctypes.c_int32),
        ("optim_balance", ctypes.c_int32),
        ("optim_chunk", ctypes.c_int32),
        ("pso_swarm", ctypes.c_uint32),
        ("pso_iters", ctypes.c_uint32),
        ("pso_stagnation", ctypes.c_uint32),
        ("pso_restart", ctypes.c_uint32),
        ("pso_p_personal", ctypes.c_double),
        ("pso_p_global", ctypes.c_double),
        ("pso_inertia", ctypes.c_double),
        ("pso_kick", ctypes.c_double),
    ]


@dataclass
class Cfg:
    """Python view of the reference PipelineConfig (config.hpp:17-36) with the
    reference defaults (README.md:137-165)."""

    dataset_size: int
    num_epochs: int
    num_nodes: int
    local_batch: int
    seed: int = 0
    buffer_capacity: int = 1
    drop_last: bool = True
    policy: str = "clairvoyant"
    graph_mode: str = "global"
    chunk_threshold: int = 15
    chunk_insert_redundant: bool = False
    optim_order: bool = True
    optim_remap: bool = True
    optim_balance: bool = True
    optim_chunk: bool = True
    pso_swarm: int = 32
    pso_iters: int = 500
    pso_stagnation: int = 100
    pso_restart: int = 20
    pso_p_personal: float = 0.5
    pso_p_global: float = 0.5
    pso_inertia: float = 0.5
    pso_kick: float = 1.0

    @property
    def B(self) -> int:
        return self.num_nodes * self.local_batch

    @property
    def steps(self) -> int:
        if self.B == 0:
            return 0
        return self.dataset_size // self.B if self.drop_last else -(-self.dataset_size // self.B)

    @property
    def keep(self) -> int:
        return self.steps * self.B if self.drop_last else self.dataset_size

    def to_c(self) -> OrConfig:
        c = OrConfig()
        c.dataset_size = self.dataset_size
        c.num_epochs = self.num_epochs
        c.num_nodes = self.num_nodes
        c.local_batch = self.local_batch
        c.seed = self.seed
        c.drop_last = int(self.drop_last)
        c.policy = 0 if self.policy == "clairvoyant" else 1
        c.buffer_capacity = self.buffer_capacity
        c.graph_mode = 0 if self.graph_mode == "global" else 1
        c.insert_redundant = int(self.chunk_insert_redundant)
        c.chunk_threshold = self.chunk_threshold
        c.optim_order = int(self.optim_order)
        c.optim_remap = int(self.optim_remap)
        c.optim_balance = int(self.optim_balance)
        c.optim_chunk = int(self.optim_chunk)
        c.pso_swarm = self.pso_swarm
        c.pso_iters = self.pso_iters
        c.pso_stagnation = self.pso_stagnation
        c.pso_restart = self.pso_restart
        c.pso_p_personal = self.pso_p_personal
        c.pso_p_global = self.pso_p_global
        c.pso_inertia = self.pso_inertia
        c.pso_kick = self.pso_kick
        return c

    def kv(self) -> list[str]:
        """key=value entries in the reference config vocabulary (config.cpp)."""
        b = lambda v: "1" if v else "0"  # noqa: E731
        return [
            f"dataset_size={self.dataset_size}", f"num_epochs={self.num_epochs}",
            f"num_nodes={self.num_nodes}", f"local_batch={self.local_batch}",
            f"seed={self.seed}", f"drop_last={b(self.drop_last)}",
            f"buffer_capacity={self.buffer_capacity}", f"policy={self.policy}",
            f"graph_mode={'global' if self.graph_mode == 'global' else 'pernode'}",
            f"chunk_threshold={self.chunk_threshold}",
            f"chunk_insert_redundant={b(self.chunk_insert_redundant)}",
            f"optim_order={b(self.optim_order)}", f"optim_remap={b(self.optim_remap)}",
            f"optim_balance={b(self.optim_balance)}", f"optim_chunk={b(self.optim_chunk)}",
            f"pso_swarm={self.pso_swarm}", f"pso_iters={self.pso_iters}",
            f"pso_stagnation={self.pso_stagnation}", f"pso_restart={self.pso_restart}",
            f"pso_p_personal={self.pso_p_personal!r}", f"pso_p_global={self.pso_p_global!r}",
            f"pso_inertia={self.pso_inertia!r}", f"pso_kick={self.pso_kick!r}",
        ]


@dataclass
class PlanArrays:
    """Flat plan layout shared by the oracle, the reference dump and the GPU."""

    trace: np.ndarray          # u32 [E, keep]
    graph: np.ndarray          # u64 [E, E]
    order: np.ndarray          # u32 [E]
    cost: int
    hist: np.ndarray           # u64 [iters]
    iters: int
    items: np.ndarray          # u32 [E*keep]  id | HIT_BIT
    node_off: np.ndarray       # u32 [T, N+1]
    fb: np.ndarray             # u32 [T, N]
    fa: np.ndarray             # u32 [T, N]
    hits: np.ndarray | None = None     # u32 [T, N]
    misses: np.ndarray | None = None   # u32 [T, N]
    residency: np.ndarray | None = None  # u64 [T, N, 3]
    extra: dict = field(default_factory=dict)


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-C", HERE, "oracle"], check=True, capture_output=True)
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        u64, u32, i32, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        L.or_splitmix_next.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        L.or_splitmix_next.restype = u64
        L.or_generate_trace.argtypes = [u64, u32, u32, u64, u64, i32, P]
        L.or_build_reuse_graph.argtypes = [P, u32, u64, u64, u32, u64, i32, u64, i32, P]
        L.or_pso_order.argtypes = [P, u32, u32, u32, dbl, dbl, dbl, dbl, u32, u32, u64, P, P, P, P]
        L.or_brute_force_order.argtypes = [P, u32, P, P]
        L.or_remap_step.argtypes = [P, P, u64, u32, u64, i32, P, P]
        L.or_balance_step.argtypes = [P, P, u32, P]
        L.or_plan.argtypes = [ctypes.POINTER(OrConfig), P, P, P, P, P, P, P, P, P, P, P]
        L.or_simulate.argtypes = [P, P, u64, u32, u64, u64, i32, P, P]
        L.or_simulate_ex.argtypes = [P, P, u64, u32, u64, u64, i32, P, P, P, P, P]
        L.or_simulate_sequence.argtypes = [P, u64, u64, u64, i32, P]
        L.or_plan_reads.argtypes = [P, P, u64, u32, i32, u64, P, P, P, P, P]
        L.or_store_payload.argtypes = [u64, u64, u64, P]
        L.or_store_payload.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: error class {code}")
        self.code = code


def _check(rc: int, what: str):
    if rc:
        raise OracleError(rc, what)


def splitmix_stream(seed: int, n: int) -> list[int]:
    s = ctypes.c_uint64(seed)
    return [lib().or_splitmix_next(ctypes.byref(s)) for _ in range(n)]


def generate_trace(D, E, N, b, seed, drop_last=True) -> np.ndarray:
    c = Cfg(D, E, N, b, seed, drop_last=drop_last)
    out = np.zeros((E, max(c.keep, 1)), dtype=np.uint32)
    _check(lib().or_generate_trace(D, E, N, b, seed, int(drop_last), _p(out)), "generate_trace")
    return out[:, : c.keep]


def build_reuse_graph(trace: np.ndarray, D, N, b, buffer_size, mode="global", drop_last=True):
    trace = np.ascontiguousarray(trace, dtype=np.uint32)
    E, L = trace.shape
    w = np.zeros((E, E), dtype=np.uint64)
    _check(lib().or_build_reuse_graph(_p(trace), E, L, D, N, b, int(drop_last), buffer_size,
                                      0 if mode == "global" else 1, _p(w)), "build_reuse_graph")
    return w


def pso_order(w: np.ndarray, seed: int, swarm=32, iters=500, p_personal=0.5, p_global=0.5,
              inertia=0.5, kick=1.0, stagnation=100, restart=20):
    w = np.ascontiguousarray(w, dtype=np.uint64)
    E = w.shape[0]
    order = np.zeros(E, dtype=np.uint32)
    cost = np.zeros(1, dtype=np.uint64)
    hist = np.zeros(max(iters, 1), dtype=np.uint64)
    n = np.zeros(1, dtype=np.uint32)
    _check(lib().or_pso_order(_p(w), E, swarm, iters, p_personal, p_global, inertia, kick,
                              stagnation, restart, seed, _p(order), _p(cost), _p(hist), _p(n)),
           "pso_order")
    return order, int(cost[0]), hist[: int(n[0])], int(n[0])


def brute_force_order(w: np.ndarray):
    w = np.ascontiguousarray(w, dtype=np.uint64)
    E = w.shape[0]
    order = np.zeros(max(E, 1), dtype=np.uint32)
    cost = np.zeros(1, dtype=np.uint64)
    _check(lib().or_brute_force_order(_p(w), E, _p(order), _p(cost)), "brute_force_order")
    return order[:E], int(cost[0])


def remap_step(holders, batch, N, b, slice_=False):
    holders = np.ascontiguousarray(holders, dtype=np.uint64)
    batch = np.ascontiguousarray(batch, dtype=np.uint32)
    items = np.zeros(max(len(batch), 1), dtype=np.uint32)
    off = np.zeros(N + 1, dtype=np.uint32)
    _check(lib().or_remap_step(_p(holders), _p(batch), len(batch), N, b, int(slice_), _p(items),
                               _p(off)), "remap_step")
    return items[: off[N]], off


def balance_step(items, node_off):
    items = np.array(items, dtype=np.uint32)
    off = np.array(node_off, dtype=np.uint32)
    moves = np.zeros(1, dtype=np.uint64)
    _check(lib().or_balance_step(_p(items), _p(off), len(off) - 1, _p(moves)), "balance_step")
    return items, off, int(moves[0])


def plan(cfg: Cfg, residency=False) -> PlanArrays:
    E, N, T = cfg.num_epochs, cfg.num_nodes, cfg.num_epochs * cfg.steps
    trace = np.zeros((E, max(cfg.keep, 1)), dtype=np.uint32)
    graph = np.zeros((E, E), dtype=np.uint64)
    order = np.zeros(E, dtype=np.uint32)
    cost = np.zeros(1, dtype=np.uint64)
    hist = np.zeros(max(cfg.pso_iters, 1), dtype=np.uint64)
    n_it = np.zeros(1, dtype=np.uint32)
    items = np.zeros(max(E * cfg.keep, 1), dtype=np.uint32)
    off = np.zeros((T, N + 1), dtype=np.uint32)
    fb = np.zeros((T, N), dtype=np.uint32)
    fa = np.zeros((T, N), dtype=np.uint32)
    res = np.zeros((T, N, 3), dtype=np.uint64) if residency else None
    c = cfg.to_c()
    _check(lib().or_plan(ctypes.byref(c), _p(trace), _p(graph), _p(order), _p(cost), _p(hist),
                         _p(n_it), _p(items), _p(off), _p(fb), _p(fa),
                         _p(res) if res is not None else None), "plan")
    it = int(n_it[0]) if cfg.optim_order else 0
    return PlanArrays(trace[:, : cfg.keep], graph, order, int(cost[0]), hist[:it], it,
                      items[: E * cfg.keep], off, fb, fa, residency=res)


def simulate(items, node_off, N, D, C, policy="clairvoyant"):
    items = np.ascontiguousarray(items, dtype=np.uint32)
    node_off = np.ascontiguousarray(node_off, dtype=np.uint32).reshape(-1, N + 1)
    T = node_off.shape[0]
    hits = np.zeros((T, N), dtype=np.uint32)
    misses = np.zeros((T, N), dtype=np.uint32)
    _check(lib().or_simulate(_p(items), _p(node_off), T, N, D, C,
                             0 if policy == "clairvoyant" else 1, _p(hits), _p(misses)), "simulate")
    return hits, misses


def simulate_redundant(items, node_off, N, D, C, rstart, rend, rcount, policy="clairvoyant"):
    """simulate_plan(..., insert_redundant=true) (buffer.cpp:224-238); the
    reads of list (g, k) sit at its item offsets (plan_reads layout)."""
    items = np.ascontiguousarray(items, dtype=np.uint32)
    node_off = np.ascontiguousarray(node_off, dtype=np.uint32).reshape(-1, N + 1)
    rstart = np.ascontiguousarray(rstart, dtype=np.uint32)
    rend = np.ascontiguousarray(rend, dtype=np.uint32)
    rcount = np.ascontiguousarray(rcount, dtype=np.uint32)
    T = node_off.shape[0]
    hits = np.zeros((T, N), dtype=np.uint32)
    misses = np.zeros((T, N), dtype=np.uint32)
    _check(lib().or_simulate_ex(_p(items), _p(node_off), T, N, D, C, 0 if policy == "clairvoyant" else 1,
                                _p(rstart), _p(rend), _p(rcount), _p(hits), _p(misses)), "simulate")
    return hits, misses


def plan_reads(items, node_off, N, chunked=True, threshold=15):
    """chunking.cpp:9-33 / pipeline.cpp:21-28 reads of every (step, node) list."""
    items = np.ascontiguousarray(items, dtype=np.uint32)
    node_off = np.ascontiguousarray(node_off, dtype=np.uint32).reshape(-1, N + 1)
    T = node_off.shape[0]
    rs = np.zeros(max(items.size, 1), np.uint32)
    re_ = np.zeros(max(items.size, 1), np.uint32)
    cnt, need, red = (np.zeros((T, N), np.uint32) for _ in range(3))
    _check(lib().or_plan_reads(_p(items), _p(node_off), T, N, int(chunked), threshold, _p(rs), _p(re_),
                               _p(cnt), _p(need), _p(red)), "plan_reads")
    return rs[: items.size], re_[: items.size], cnt, need, red


def simulate_sequence(seq, C, policy="clairvoyant"):
    seq = np.ascontiguousarray(seq, dtype=np.uint32)
    D = int(seq.max()) + 1 if len(seq) else 1
    m = np.zeros(1, dtype=np.uint64)
    _check(lib().or_simulate_sequence(_p(seq), len(seq), D, C, 0 if policy == "clairvoyant" else 1,
                                      _p(m)), "simulate_sequence")
    return int(m[0])


def store_payload(fill_seed: int, offset: int, n: int) -> np.ndarray:
    out = np.zeros(max(n, 1), dtype=np.uint8)
    lib().or_store_payload(fill_seed, offset, n, _p(out))
    return out[:n]


def compact_reads(rstart, rend, rcount, node_off, N):
    """The valid (start, end) pairs of every (step, node) list in plan order
    (list (g, k)'s reads sit at its item offsets): the layout-independent form
    the full-size goldens hash (tools/make_goldens.py)."""
    node_off = np.asarray(node_off).reshape(-1, N + 1).astype(np.int64)
    base = np.concatenate([[0], np.cumsum(node_off[:, N])[:-1]])
    lo = (base[:, None] + node_off[:, :N]).ravel()
    cnt = np.asarray(rcount).reshape(-1).astype(np.int64)
    idx = np.repeat(lo, cnt) + (np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt))
    return np.stack([np.asarray(rstart)[idx], np.asarray(rend)[idx]], axis=1).astype(np.uint32)


# ------------------------------------------------------- compiled reference --
def ref_available() -> bool:
    return os.path.exists(REF_DUMP)


def ref_text(cfg: Cfg, extra: tuple[str, ...] = ()) -> dict:
    """The UNMODIFIED reference's write_trace/write_graph/write_plan files of a
    plan_schedule run, its write_metrics (metrics.csv of the configured pass)
    and total_barrier_cost / total_io_cost ("%.6f %.6f"): {"trace", "graph",
    "plan", "metrics", "costs"} -> bytes."""
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([REF_DUMP, "text", d, *cfg.kv(), *extra], check=True, capture_output=True)
        out = {k: open(os.path.join(d, k + ".txt"), "rb").read() for k in ("trace", "graph", "plan", "costs",
                                                                               "costs_exact")}
        out["metrics"] = open(os.path.join(d, "metrics.csv"), "rb").read()
        return out


def ref_run_pipeline(d: str) -> dict:
    """The reference's run_pipeline artifacts (test_pipeline.cpp's small
    config) written into d: {file name: bytes}."""
    subprocess.run([REF_DUMP, "runpipe", d], check=True, capture_output=True)
    return {n: open(os.path.join(d, n), "rb").read() for n in sorted(os.listdir(d))}


def ref_read(kind: str, data: bytes) -> tuple[int, str]:
    """The reference's read_trace/read_graph/read_plan on `data`: (0, "") or
    (error class, message)."""
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "in.txt")
        with open(p, "wb") as f:
            f.write(data)
        out = subprocess.run([REF_DUMP, "read", kind, p], check=True, capture_output=True,
                             text=True).stdout.rstrip("\n")
    if out.startswith("ok"):
        return 0, ""
    _, code, msg = out.split(" ", 2)
    return int(code), msg


def ref_plan(cfg: Cfg) -> PlanArrays:
    """Run the UNMODIFIED reference plan_schedule + simulate_plan."""
    E, N, T = cfg.num_epochs, cfg.num_nodes, cfg.num_epochs * cfg.steps
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([REF_DUMP, "plan", d, *cfg.kv()], check=True, capture_output=True)
        rd = lambda n, t: np.fromfile(os.path.join(d, n), dtype=t)  # noqa: E731
        hist = rd("hist.u64", np.uint64) if os.path.exists(os.path.join(d, "hist.u64")) else np.zeros(0, np.uint64)
        iters = int(rd("iters.u32", np.uint32)[0]) if os.path.exists(os.path.join(d, "iters.u32")) else 0
        resp = os.path.join(d, "residency.u64")
        return PlanArrays(
            trace=rd("trace.u32", np.uint32).reshape(E, cfg.keep),
            graph=rd("graph.u64", np.uint64).reshape(E, E),
            order=rd("order.u32", np.uint32),
            cost=int(rd("cost.u64", np.uint64)[0]),
            hist=hist, iters=iters,
            items=rd("items.u32", np.uint32),
            node_off=rd("nodeoff.u32", np.uint32).reshape(T, N + 1),
            fb=rd("fb.u32", np.uint32).reshape(T, N),
            fa=rd("fa.u32", np.uint32).reshape(T, N),
            hits=rd("hits.u32", np.uint32).reshape(T, N),
            misses=rd("misses.u32", np.uint32).reshape(T, N),
            residency=np.fromfile(resp, dtype=np.uint64).reshape(T, N, 3) if os.path.exists(resp) else None,
            extra={n: rd(n + ".u32", np.uint32) for n in ("rstart", "rend", "rcount", "rneed", "rred")},
        )


def ref_simulate(items, node_off, N, D, steps_per_epoch, C, policy="clairvoyant"):
    node_off = np.ascontiguousarray(node_off, dtype=np.uint32)
    T = node_off.size // (N + 1)
    with tempfile.TemporaryDirectory() as d:
        np.ascontiguousarray(items, dtype=np.uint32).tofile(os.path.join(d, "items.u32"))
        node_off.tofile(os.path.join(d, "nodeoff.u32"))
        subprocess.run([REF_DUMP, "simulate", d, str(N), str(D), str(steps_per_epoch), str(C),
                        policy], check=True, capture_output=True)
        return (np.fromfile(os.path.join(d, "hits.u32"), dtype=np.uint32).reshape(T, N),
                np.fromfile(os.path.join(d, "misses.u32"), dtype=np.uint32).reshape(T, N))


def ref_time(cfg: Cfg, reps: int = 1) -> dict:
    out = subprocess.run([REF_DUMP, "time", str(reps), *cfg.kv()], check=True,
                         capture_output=True, text=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def ref_store_file(path: str, count: int, size: int, seed: int) -> None:
    """The UNMODIFIED reference create_store writes `path` (header + payload)."""
    subprocess.run([REF_DUMP, "storefile", str(path), str(count), str(size), str(seed)], check=True,
                   capture_output=True)


def ref_store(count: int, size: int, seed: int) -> np.ndarray:
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "payload")
        subprocess.run([REF_DUMP, "store", p, str(count), str(size), str(seed)], check=True,
                       capture_output=True)
        return np.fromfile(p, dtype=np.uint8)
