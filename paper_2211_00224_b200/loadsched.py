"""Python mirror of the reference ``loadsched`` planner API, backed by the
sm_100a kernels through the C ABI (include/lsg.h).

Names, argument meaning and error classes follow the reference headers
(/root/reference/proj/include/loadsched/*.hpp, cited per function) so parity
tests read like the reference's own tests. Tensors live on the current CUDA
device; uint32 data is carried in int32 tensors (same bits) and uint64 in
int64 tensors. Every call goes to the CUDA library; there is no CPU path.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import HIT_BIT, NEVER, LsgConfig, LsgError, LsgPlanOut, LsgShape, check, lib

__all__ = [
    "TraceConfig", "PsoParams", "PipelineConfig", "AccessTrace", "ReuseGraph", "EpochOrder",
    "PsoResult", "SchedulePlan", "PlanOutput", "SimResult", "generate_trace", "build_reuse_graph",
    "pso_order", "build_reuse_graph_rows", "identity_order", "plan_schedule", "plan_schedule_host", "plan_host_buffers", "baseline_config", "simulate_plan",
    "store_fill", "gather", "batch_fetch", "StepFetcher", "StoreHeader", "Store", "create_store",
    "STORE_HEADER_BYTES", "DEFAULT_STORE_BUDGET", "format_trace", "write_trace_file", "read_trace",
    "read_trace_file", "format_graph", "write_graph_file", "read_graph", "read_graph_file", "format_plan",
    "write_plan_file", "read_plan", "read_plan_file", "Error", "ConfigError", "ValidationError", "CapabilityError",
    "StorageError", "InternalError", "HIT_BIT", "NEVER", "brute_force_order", "remap_step", "slice_step",
    "remap_epoch", "balance_step", "Read", "ChunkPlan", "plan_chunks", "K_NEVER_USED", "Buffer", "make_buffer",
    "simulate_sequence", "optimal_miss_oracle", "CostModel", "policy_name", "total_barrier_cost",
    "total_io_cost", "format_metrics", "write_metrics_file", "to_host", "HostRows", "FetchJob", "MissStream",
]


# --------------------------------------------------------------- errors --
# errors.hpp:10-46 — one class per ErrorClass, all subclasses of LsgError.
class Error(LsgError):
    pass


class ConfigError(Error):
    pass


class ValidationError(Error):
    pass


class CapabilityError(Error):
    pass


class StorageError(Error):
    pass


class InternalError(Error):
    pass


_BY_CODE = {_lib.CONFIG: ConfigError, _lib.VALIDATION: ValidationError,
            _lib.CAPABILITY: CapabilityError, _lib.STORAGE: StorageError,
            _lib.INTERNAL: InternalError}


def _check(rc: int) -> None:
    if rc != 0:
        raise _BY_CODE.get(rc, Error)(rc, lib().lsg_last_error().decode())


def _policy_code(policy: str) -> int:
    """config.cpp:71-74: anything but the two names is a ConfigError."""
    if policy == "clairvoyant":
        return 0
    if policy == "lru":
        return 1
    raise ConfigError(2, "policy must be clairvoyant or lru")


def _mode_code(mode: str) -> int:
    """config.cpp:75-78"""
    if mode == "global":
        return 0
    if mode == "pernode":
        return 1
    raise ConfigError(2, "graph_mode must be global or pernode")


# --------------------------------------------------------------- config --
@dataclass
class TraceConfig:
    """trace.hpp:15-27"""

    dataset_size: int = 0
    num_epochs: int = 0
    num_nodes: int = 0
    local_batch: int = 0
    seed: int = 0
    drop_last: bool = True

    def global_batch(self) -> int:
        return self.num_nodes * self.local_batch

    def steps_per_epoch(self) -> int:  # trace.cpp:12-16
        B = self.global_batch()
        if B == 0:
            return 0
        return self.dataset_size // B if self.drop_last else -(-self.dataset_size // B)

    def keep(self) -> int:
        return self.steps_per_epoch() * self.global_batch() if self.drop_last else self.dataset_size


@dataclass
class PsoParams:
    """epoch_order.hpp:18-29"""

    swarm_size: int = 32
    max_iters: int = 500
    p_personal: float = 0.5
    p_global: float = 0.5
    inertia: float = 0.5
    kick: float = 1.0
    stagnation_limit: int = 100
    restart_limit: int = 20
    seed: int = 0


@dataclass
class PipelineConfig:
    """config.hpp:17-36 (cost-model fields omitted: they never reach the path)."""

    trace: TraceConfig = field(default_factory=TraceConfig)
    buffer_capacity: int = 0
    policy: str = "clairvoyant"       # "clairvoyant" | "lru"
    graph_mode: str = "global"        # "global" | "pernode"
    chunk_threshold: int = 15
    chunk_insert_redundant: bool = False
    pso: PsoParams = field(default_factory=PsoParams)
    optim_order: bool = True
    optim_remap: bool = True
    optim_balance: bool = True
    optim_chunk: bool = True

    def to_c(self) -> LsgConfig:
        c = LsgConfig()
        t = self.trace
        c.dataset_size, c.num_epochs, c.num_nodes = t.dataset_size, t.num_epochs, t.num_nodes
        c.local_batch, c.seed, c.drop_last = t.local_batch, t.seed, int(t.drop_last)
        c.policy = _policy_code(self.policy)
        c.buffer_capacity = self.buffer_capacity
        c.graph_mode = _mode_code(self.graph_mode)
        c.insert_redundant = int(self.chunk_insert_redundant)
        c.chunk_threshold = self.chunk_threshold
        c.optim_order, c.optim_remap = int(self.optim_order), int(self.optim_remap)
        c.optim_balance, c.optim_chunk = int(self.optim_balance), int(self.optim_chunk)
        p = self.pso
        c.pso_swarm, c.pso_iters, c.pso_stagnation, c.pso_restart = (
            p.swarm_size, p.max_iters, p.stagnation_limit, p.restart_limit)
        c.pso_p_personal, c.pso_p_global, c.pso_inertia, c.pso_kick = (
            p.p_personal, p.p_global, p.inertia, p.kick)
        return c

    def shape(self) -> LsgShape:
        sh = LsgShape()
        c = self.to_c()
        _check(lib().lsg_shape_of(ctypes.byref(c), ctypes.byref(sh)))
        return sh

    def validate(self) -> None:  # config.cpp:11-22
        self.shape()


# ---------------------------------------------------------------- types --
@dataclass
class AccessTrace:
    """trace.hpp:33-38; epochs: int32 [E, keep] on device (uint32 ids)."""

    config: TraceConfig
    epochs: torch.Tensor


@dataclass
class ReuseGraph:
    """reuse_graph.hpp:23-35; weights: int64 [E, E] on device."""

    num_epochs: int
    buffer_size: int
    mode: str
    weights: torch.Tensor


@dataclass
class EpochOrder:
    order: torch.Tensor  # int32 [E]
    cost: int


@dataclass
class PsoResult:
    """epoch_order.hpp:39-43"""

    best: EpochOrder
    history: torch.Tensor  # int64 [iterations]
    iterations: int


@dataclass
class SchedulePlan:
    """plan.hpp:33-53 in flat device layout: steps in execution order; step g's
    node k list is items[base_g + node_off[g,k] : base_g + node_off[g,k+1]]
    with base_g = sum of earlier steps' lengths; bit 31 of an item = hit tag."""

    dataset_size: int
    num_nodes: int
    local_batch: int
    steps_per_epoch: int
    order: EpochOrder
    items: torch.Tensor         # int32 [E*keep]
    node_off: torch.Tensor      # int32 [T, N+1]
    fetches_before: torch.Tensor  # int32 [T, N]
    fetches_after: torch.Tensor   # int32 [T, N]
    # StepPlan.reads (pipeline.cpp:83-88): list (g, k)'s reads at its item
    # offsets (start == end: Single read), counts / needed / redundant [T, N]
    read_start: torch.Tensor | None = None
    read_end: torch.Tensor | None = None
    read_count: torch.Tensor | None = None
    read_needed: torch.Tensor | None = None
    read_redundant: torch.Tensor | None = None
    chunk_threshold: int = 0    # plan.hpp: the threshold the reads were cut with (0: no chunking)


@dataclass
class PlanOutput:
    """pipeline.hpp:17-22"""

    trace: AccessTrace
    graph: ReuseGraph
    pso: PsoResult | None
    plan: SchedulePlan


@dataclass
class SimResult:
    """buffer.hpp:106-111; rows as [T, N] tensors (execution order, nodes ascending)."""

    hits: torch.Tensor
    misses: torch.Tensor
    total_hits: int
    total_misses: int
    slots: torch.Tensor | None = None
    policy: str = "clairvoyant"  # the replay's policy (metrics.csv labels its rows with it)


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def to_host(t: torch.Tensor) -> torch.Tensor:
    """Device -> host copy through PINNED memory on the current stream, then a
    sync of that stream only. (A copy into pageable memory is staged by the
    driver and can wait for kernels of OTHER streams: a replay's readback sat
    behind a concurrent planner's persistent kernel.)"""
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2211_00224_b200 requires a CUDA (sm_100a) device")
    return torch.device("cuda", torch.cuda.current_device())


# ------------------------------------------------------------- functions --
def generate_trace(config: TraceConfig) -> AccessTrace:
    """trace.hpp:40 / trace.cpp:26-43 — K1 on device."""
    pc = PipelineConfig(trace=config, buffer_capacity=1)
    c = pc.to_c()
    keep = config.keep() if config.global_batch() else 0
    out = torch.empty((max(config.num_epochs, 1), max(keep, 1)), dtype=torch.int32, device=_dev())
    _check(lib().lsg_generate_trace(ctypes.byref(c), _ptr(out), _stream()))
    return AccessTrace(config, out[: config.num_epochs, :keep])


def build_reuse_graph(trace: AccessTrace, buffer_size: int, mode: str = "global") -> ReuseGraph:
    """reuse_graph.hpp:53 / reuse_graph.cpp:77-101 — K2+K3 on device. The trace
    may repeat ids (read_trace admits it)."""
    ep = trace.epochs.contiguous()
    E, L = ep.shape
    w = torch.empty((max(E, 1), max(E, 1)), dtype=torch.int64, device=ep.device)
    cfg = trace.config
    _check(lib().lsg_build_reuse_graph(_ptr(ep), E, L, cfg.dataset_size, cfg.num_nodes,
                                       cfg.local_batch, int(cfg.drop_last), buffer_size,
                                       _mode_code(mode), _ptr(w), _stream()))
    return ReuseGraph(E, buffer_size, mode, w[:E, :E])


def build_reuse_graph_rows(trace: AccessTrace, buffer_size: int, mode: str, row_begin: int,
                           row_end: int) -> torch.Tensor:
    """Rows [row_begin, row_end) of build_reuse_graph's weights (int64
    [row_end - row_begin, E] on device): the row block one GPU computes in the
    multi-GPU row sharding of K3 (parallel.sharded_reuse_graph)."""
    ep = trace.epochs.contiguous()
    E, L = ep.shape
    rows = torch.empty((max(row_end - row_begin, 0), E), dtype=torch.int64, device=ep.device)
    cfg = trace.config
    _check(lib().lsg_build_reuse_graph_rows(_ptr(ep), E, L, cfg.dataset_size, cfg.num_nodes, cfg.local_batch,
                                            int(cfg.drop_last), buffer_size, _mode_code(mode),
                                            row_begin, row_end, _ptr(rows) if rows.numel() else None,
                                            _stream()))
    return rows


def pso_order(graph: ReuseGraph, params: PsoParams) -> PsoResult:
    """epoch_order.hpp:60 / epoch_order.cpp:121-221 — K4, bit-exact."""
    E = graph.num_epochs
    dev = graph.weights.device
    order = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    cost = torch.empty(1, dtype=torch.int64, device=dev)
    hist = torch.empty(max(params.max_iters, 1), dtype=torch.int64, device=dev)
    iters = torch.empty(1, dtype=torch.int32, device=dev)
    w = graph.weights.contiguous()
    _check(lib().lsg_pso_order(_ptr(w), E, params.swarm_size, params.max_iters, params.p_personal,
                               params.p_global, params.inertia, params.kick,
                               params.stagnation_limit, params.restart_limit, params.seed,
                               _ptr(order), _ptr(cost), _ptr(hist), _ptr(iters), _stream()))
    n = int(iters.item())
    return PsoResult(EpochOrder(order[:E], int(cost.item())), hist[:n], n)


def identity_order(graph: ReuseGraph) -> EpochOrder:
    """epoch_order.hpp:63"""
    E = graph.num_epochs
    if E == 0:
        raise ValidationError(_lib.VALIDATION, "identity_order: empty graph")
    idx = torch.arange(E, device=graph.weights.device)
    cost = int(graph.weights[idx[:-1], idx[1:]].sum().item()) if E > 1 else 0
    return EpochOrder(idx.to(torch.int32), cost)


def brute_force_order(graph: ReuseGraph) -> EpochOrder:
    """epoch_order.hpp:35-38 / epoch_order.cpp:32-52 — one CTA over all E!
    open paths (E <= 10), ties to the lexicographically smallest order."""
    E = graph.num_epochs
    dev = graph.weights.device
    order = torch.empty(max(E, 1), dtype=torch.int32, device=dev)
    cost = torch.empty(1, dtype=torch.int64, device=dev)
    w = graph.weights.contiguous()
    _check(lib().lsg_brute_force_order(_ptr(w), E, _ptr(order), _ptr(cost), _stream()))
    return EpochOrder(order[:E], int(cost.item()))


def _host_u32(a, what: str) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1))
    if a.size and (a.min() < 0 or a.max() >= 1 << 31):
        raise CapabilityError(_lib.CAPABILITY, f"{what}: sample ids must be < 2^31 on device")
    return a.astype(np.uint32)


def _np_ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


def _locality(buffers, batch, local_batch: int, slice_: bool):
    N = len(buffers)
    res = [_host_u32(sorted(s), "remap_step") for s in buffers]
    roff = np.zeros(N + 1, dtype=np.uint64)
    if N:
        roff[1:] = np.cumsum([r.size for r in res])
    rids = np.concatenate(res) if N and roff[N] else np.zeros(1, dtype=np.uint32)
    ids = _host_u32(batch, "remap_step")
    items = np.zeros(ids.size + 1, dtype=np.uint32)
    off = np.zeros(N + 1, dtype=np.uint32)
    _check(lib().lsg_remap_step(_np_ptr(roff), _np_ptr(rids), N, _np_ptr(ids), ids.size, local_batch,
                                int(slice_), _np_ptr(items), _np_ptr(off), None))
    return items[: off[N]], off


def remap_step(buffers, batch, local_batch: int):
    """locality.hpp:23-25 / locality.cpp:7-39 — one step of the device step
    loop against explicit residency sets (buffers: one id collection per node).
    Returns (items uint32 with bit 31 = hit, node_off uint32 [N+1])."""
    return _locality(buffers, batch, local_batch, False)


def slice_step(buffers, batch, local_batch: int):
    """locality.hpp:36-38 / locality.cpp:56-73"""
    return _locality(buffers, batch, local_batch, True)


def remap_epoch(prev_buffers, epoch_batches, local_batch: int):
    """locality.hpp:30-32: every step against one fixed residency snapshot."""
    return [remap_step(prev_buffers, b, local_batch) for b in epoch_batches]


def balance_step(items, node_off):
    """balance.hpp:20 / balance.cpp:10-39 — closed-form move table on the
    device. Returns (items, node_off, moves)."""
    it = np.array(items, dtype=np.uint32).reshape(-1)
    off = np.array(node_off, dtype=np.uint32).reshape(-1)
    buf = np.zeros(it.size + 1, dtype=np.uint32)
    buf[: it.size] = it
    moves = np.zeros(1, dtype=np.uint64)
    _check(lib().lsg_balance_step(_np_ptr(buf), _np_ptr(off), max(off.size - 1, 0), _np_ptr(moves), None))
    return buf[: it.size], off, int(moves[0])


@dataclass
class Read:
    """chunking.hpp:13-22"""

    kind: str  # "single" | "chunk"
    start: int
    end: int

    def span(self) -> int:
        return self.end - self.start + 1


@dataclass
class ChunkPlan:
    reads: list
    needed: int
    redundant: int


def plan_chunks(fetch_ids, threshold: int) -> ChunkPlan:
    """chunking.hpp:23-30 / chunking.cpp:9-33 — the device read planner on one list."""
    ids = _host_u32(fetch_ids, "plan_chunks")
    rs = np.zeros(ids.size + 1, dtype=np.uint32)
    re = np.zeros(ids.size + 1, dtype=np.uint32)
    meta = np.zeros(3, dtype=np.uint64)
    _check(lib().lsg_plan_chunks(_np_ptr(ids), ids.size, threshold, _np_ptr(rs), _np_ptr(re), _np_ptr(meta),
                                 None))
    n = int(meta[0])
    reads = [Read("single" if rs[i] == re[i] else "chunk", int(rs[i]), int(re[i])) for i in range(n)]
    return ChunkPlan(reads, int(meta[1]), int(meta[2]))


K_NEVER_USED = (1 << 64) - 1  # buffer.hpp:19


class Buffer:
    """buffer.hpp:21-79 — one node's buffer as device-resident state
    (lsg_buffer_*). access / insert_silent / clear / resident as in the
    reference; access_batch applies a whole sequence in one launch."""

    def __init__(self, policy: str, capacity: int):
        if capacity == 0:
            raise ValidationError(_lib.VALIDATION, "buffer capacity must be >= 1")
        self.policy, self._cap = policy, capacity
        h = ctypes.c_void_p()
        _check(lib().lsg_buffer_create(_policy_code(policy), capacity, ctypes.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().lsg_buffer_destroy(h)
            self._h = None

    def capacity(self) -> int:
        return self._cap

    def _ops(self, ids, next_use, silent: bool) -> np.ndarray:
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64).reshape(-1))
        nu = np.ascontiguousarray(np.asarray(next_use, dtype=np.uint64).reshape(-1))
        if nu.size != ids.size:
            raise ValidationError(_lib.VALIDATION, "access_batch: ids and next_use differ in length")
        hit = np.zeros(max(ids.size, 1), dtype=np.uint8)
        _check(lib().lsg_buffer_access(self._h, _np_ptr(ids), _np_ptr(nu), ids.size, int(silent), _np_ptr(hit),
                                       None))
        return hit[: ids.size].astype(bool)

    def access(self, sample_id: int, next_use: int = K_NEVER_USED) -> bool:
        return bool(self._ops([sample_id], [next_use], False)[0])

    def access_batch(self, ids, next_use) -> np.ndarray:
        return self._ops(ids, next_use, False)

    def insert_silent(self, sample_id: int, next_use: int = K_NEVER_USED) -> None:
        self._ops([sample_id], [next_use], True)

    def clear(self) -> None:
        _check(lib().lsg_buffer_clear(self._h))

    def resident(self) -> set:
        n = ctypes.c_uint64(0)
        _check(lib().lsg_buffer_resident(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(max(n.value, 1), dtype=np.uint64)
        _check(lib().lsg_buffer_resident(self._h, _np_ptr(out), n.value, ctypes.byref(n)))
        return set(int(v) for v in out[: n.value])


def make_buffer(policy: str, capacity: int) -> Buffer:
    """buffer.hpp:79"""
    return Buffer(policy, capacity)


def simulate_sequence(seq, capacity: int, policy: str = "clairvoyant") -> int:
    """buffer.hpp:83-84 / buffer.cpp:116-125 — one node through the K7 replay."""
    ids = _host_u32(seq, "simulate_sequence")
    m = ctypes.c_uint64(0)
    _check(lib().lsg_simulate_sequence(_np_ptr(ids), ids.size, capacity, _policy_code(policy),
                                       ctypes.byref(m), None))
    return m.value


def optimal_miss_oracle(seq, capacity: int) -> int:
    """buffer.hpp:88 / buffer.cpp:132-182 — exhaustive optimum (length <= 16,
    capacity 1..4) as a device DP."""
    s = np.ascontiguousarray(np.asarray(seq, dtype=np.uint64).reshape(-1))
    m = ctypes.c_uint64(0)
    _check(lib().lsg_optimal_miss_oracle(_np_ptr(s), s.size, capacity, ctypes.byref(m), None))
    return m.value


def _plan_buffers(config: PipelineConfig, dev):
    sh = config.shape()
    E, N, T = config.trace.num_epochs, config.trace.num_nodes, int(sh.total_steps)
    mk = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, device=dev)  # noqa: E731
    bufs = dict(trace=mk(sh.total_items, torch.int32), graph=mk(E * E, torch.int64),
                order=mk(E, torch.int32), cost=mk(1, torch.int64),
                hist=mk(config.pso.max_iters, torch.int64), iters=mk(1, torch.int32),
                items=mk(sh.total_items, torch.int32), node_off=mk(T * (N + 1), torch.int32),
                fetch_before=mk(T * N, torch.int32), fetch_after=mk(T * N, torch.int32),
                read_start=mk(sh.total_items, torch.int32), read_end=mk(sh.total_items, torch.int32),
                read_count=mk(T * N, torch.int32), read_needed=mk(T * N, torch.int32),
                read_redundant=mk(T * N, torch.int32))
    return sh, bufs


def _wrap_plan(config: PipelineConfig, sh, b) -> PlanOutput:
    t = config.trace
    E, N, T, keep = t.num_epochs, t.num_nodes, int(sh.total_steps), int(sh.keep)
    trace = AccessTrace(t, b["trace"][: E * keep].view(E, keep))
    graph = ReuseGraph(E, config.buffer_capacity, config.graph_mode, b["graph"][: E * E].view(E, E))
    order = EpochOrder(b["order"][:E], int(b["cost"][0]))
    pso = None
    if config.optim_order:
        n = int(b["iters"][0])
        pso = PsoResult(order, b["hist"][:n], n)
    plan = SchedulePlan(t.dataset_size, N, t.local_batch, int(sh.steps_per_epoch), order,
                        b["items"][: E * keep], b["node_off"][: T * (N + 1)].view(T, N + 1),
                        b["fetch_before"][: T * N].view(T, N), b["fetch_after"][: T * N].view(T, N),
                        b["read_start"][: E * keep], b["read_end"][: E * keep],
                        b["read_count"][: T * N].view(T, N), b["read_needed"][: T * N].view(T, N),
                        b["read_redundant"][: T * N].view(T, N),
                        config.chunk_threshold if config.optim_chunk else 0)  # pipeline.cpp:52
    return PlanOutput(trace, graph, pso, plan)


def plan_schedule(config: PipelineConfig) -> PlanOutput:
    """pipeline.hpp:27 / pipeline.cpp:32-120 — K1..K6 on device, outputs in HBM."""
    sh, b = _plan_buffers(config, _dev())
    out = LsgPlanOut(**{k: v.data_ptr() for k, v in b.items()})
    c = config.to_c()
    _check(lib().lsg_plan(ctypes.byref(c), ctypes.byref(out), _stream()))
    return _wrap_plan(config, sh, b)


def plan_host_buffers(config: PipelineConfig, pinned: bool = True) -> dict:
    """Host (pinned) output arrays for plan_schedule_host, allocated once by a
    loader and reused across plans."""
    sh = config.shape()
    E, N, T = config.trace.num_epochs, config.trace.num_nodes, int(sh.total_steps)
    mk = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, pin_memory=pinned)  # noqa: E731
    return dict(trace=mk(sh.total_items, torch.int32), graph=mk(E * E, torch.int64),
                order=mk(E, torch.int32), cost=mk(1, torch.int64),
                hist=mk(config.pso.max_iters, torch.int64), iters=mk(1, torch.int32),
                items=mk(sh.total_items, torch.int32), node_off=mk(T * (N + 1), torch.int32),
                fetch_before=mk(T * N, torch.int32), fetch_after=mk(T * N, torch.int32),
                read_start=mk(sh.total_items, torch.int32), read_end=mk(sh.total_items, torch.int32),
                read_count=mk(T * N, torch.int32), read_needed=mk(T * N, torch.int32),
                read_redundant=mk(T * N, torch.int32))


def plan_schedule_host(config: PipelineConfig, pinned: bool = True, buffers: dict | None = None) -> PlanOutput:
    """plan_schedule with host outputs through lsg_plan_host (the e2e path):
    device work plus the device->host copies of the whole plan (into
    `buffers` from plan_host_buffers when given)."""
    _dev()
    sh = config.shape()
    b = buffers if buffers is not None else plan_host_buffers(config, pinned)
    out = LsgPlanOut(**{k: v.data_ptr() for k, v in b.items()})
    c = config.to_c()
    _check(lib().lsg_plan_host(ctypes.byref(c), ctypes.byref(out), _stream()))
    return _wrap_plan(config, sh, b)


def baseline_config(config: PipelineConfig) -> PipelineConfig:
    """pipeline.cpp:122-131 — the comparison pass run_pipeline plans beside the
    optimised one: LRU buffers, identity order, slicing, no balance, no chunks."""
    import dataclasses
    return dataclasses.replace(config, policy="lru", optim_order=False, optim_remap=False,
                               optim_balance=False, optim_chunk=False, chunk_insert_redundant=False)


def simulate_plan(plan: SchedulePlan, capacity: int, policy: str = "clairvoyant",
                  node_range: tuple[int, int] | None = None, want_slots: bool = False,
                  insert_redundant: bool = False) -> SimResult:
    """buffer.hpp:117-118 / buffer.cpp:183-247 — K7 per-rank replay. node_range
    restricts the replay to ranks [k0, k1) (multi-GPU sharding). With
    insert_redundant the plan's chunk reads' unrequested ids are inserted
    silently after each list (clairvoyant policy, no slots)."""
    N = plan.num_nodes
    T = plan.node_off.shape[0]
    k0, k1 = node_range if node_range is not None else (0, N)
    dev = plan.items.device
    hits = torch.zeros((T, N), dtype=torch.int32, device=dev)
    misses = torch.zeros((T, N), dtype=torch.int32, device=dev)
    slots = torch.empty(max(plan.items.numel(), 1), dtype=torch.int32, device=dev) if want_slots else None
    pol = _policy_code(policy)
    if insert_redundant:
        if plan.read_start is None:
            raise ValidationError(3, "simulate_plan: insert_redundant needs the plan's reads")
        _check(lib().lsg_simulate_ex(_ptr(plan.items.contiguous()), _ptr(plan.node_off.contiguous()), T, N,
                                     plan.dataset_size, capacity, pol, 1, _ptr(plan.read_start),
                                     _ptr(plan.read_end), _ptr(plan.read_count), k0, k1, _ptr(hits),
                                     _ptr(misses), _ptr(slots), _stream()))
    else:
        _check(lib().lsg_simulate(_ptr(plan.items.contiguous()), _ptr(plan.node_off.contiguous()), T, N,
                                  plan.dataset_size, capacity, pol, k0, k1, _ptr(hits), _ptr(misses),
                                  _ptr(slots), _stream()))
    tot = to_host(torch.stack([hits.sum(dtype=torch.int64), misses.sum(dtype=torch.int64)]))
    return SimResult(hits, misses, int(tot[0]), int(tot[1]), slots[: plan.items.numel()] if slots is not None else None,
                     policy_name(policy))


def store_fill(ids: torch.Tensor, sample_bytes: int, fill_seed: int,
               out: torch.Tensor | None = None) -> torch.Tensor:
    """K9: rows = Store::read_one(ids[r]) payload (store.cpp:70-80)."""
    ids = ids.to(torch.int32).contiguous()
    n = ids.numel()
    if out is None:
        out = torch.empty((n, sample_bytes), dtype=torch.uint8, device=ids.device)
    _check(lib().lsg_store_fill(_ptr(ids), n, sample_bytes, fill_seed, _ptr(out), _stream()))
    return out


def gather(buf: torch.Tensor, slots: torch.Tensor, sample_bytes: int,
           out: torch.Tensor | None = None) -> torch.Tensor:
    """K8: out row r = buf row slots[r] (the HBM-buffer batch fetch)."""
    slots = slots.to(torch.int32).contiguous()
    n = slots.numel()
    if out is None:
        out = torch.empty((n, sample_bytes), dtype=torch.uint8, device=buf.device)
    _check(lib().lsg_gather(_ptr(buf), _ptr(slots), n, sample_bytes, _ptr(out), _stream()))
    return out


def batch_fetch(buf: torch.Tensor, ids: torch.Tensor, slots: torch.Tensor, sample_bytes: int,
                fill_seed: int, out: torch.Tensor) -> torch.Tensor:
    """K8+K9 loading phase of one node list: hits gathered from their HBM slots,
    misses written from storage (synthetic Store payload) into the batch and
    into their new slot (lsg_batch_fetch)."""
    n = ids.numel()
    _check(lib().lsg_batch_fetch(_ptr(buf), _ptr(ids), _ptr(slots), n, sample_bytes, fill_seed,
                                 _ptr(out), _stream()))
    return out


# -------------------------------------------------------------- artifacts --
# trace.cpp:72-162, reuse_graph.cpp:103-140, plan.cpp:44-227. Writers format on
# the GPU (lsg_format_*), readers accept exactly the reference's grammar.
def _two_call(fn, *args) -> bytes:
    n = ctypes.c_uint64(0)
    _check(fn(*args, None, 0, ctypes.byref(n), _stream()))
    buf = ctypes.create_string_buffer(max(1, n.value))
    _check(fn(*args, buf, n.value, ctypes.byref(n), _stream()))
    return buf.raw[: n.value]


def _write(path, data: bytes) -> None:
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise StorageError(6, f"cannot open for writing: {path}") from e


def _read(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise StorageError(6, f"cannot open for reading: {path}") from e


def format_trace(trace: AccessTrace) -> bytes:
    """write_trace (trace.cpp:72-84)."""
    c = trace.config
    ep = trace.epochs.contiguous()
    return _two_call(lib().lsg_format_trace, _ptr(ep), c.dataset_size, c.num_epochs, c.num_nodes, c.local_batch,
                     c.seed, int(c.drop_last), ep.shape[1] if ep.dim() == 2 else 0)


def write_trace_file(path, trace: AccessTrace) -> None:
    _write(path, format_trace(trace))


def read_trace(text) -> AccessTrace:
    """read_trace (trace.cpp:103-147): ids land on the device."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = _lib.LsgTraceText()
    _check(lib().lsg_parse_trace(data, len(data), ctypes.byref(h), None, 0))
    n = h.num_epochs * h.keep
    ids = torch.empty(max(n, 1), dtype=torch.int32)
    _check(lib().lsg_parse_trace(data, len(data), ctypes.byref(h), ctypes.c_void_p(ids.data_ptr()), n))
    cfg = TraceConfig(h.dataset_size, h.num_epochs, h.num_nodes, h.local_batch, h.seed, bool(h.drop_last))
    return AccessTrace(cfg, ids[:n].view(h.num_epochs, h.keep).to(_dev()))


def read_trace_file(path) -> AccessTrace:
    return read_trace(_read(path))


def format_graph(graph: ReuseGraph) -> bytes:
    """write_graph (reuse_graph.cpp:103-112)."""
    return _two_call(lib().lsg_format_graph, _ptr(graph.weights.contiguous()), graph.num_epochs)


def write_graph_file(path, graph: ReuseGraph) -> None:
    _write(path, format_graph(graph))


def read_graph(text) -> ReuseGraph:
    """read_graph (reuse_graph.cpp:114-128)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    E = ctypes.c_uint32(0)
    _check(lib().lsg_parse_graph(data, len(data), ctypes.byref(E), None, 0))
    w = torch.empty(max(E.value * E.value, 1), dtype=torch.int64)
    _check(lib().lsg_parse_graph(data, len(data), ctypes.byref(E), ctypes.c_void_p(w.data_ptr()),
                                 E.value * E.value))
    return ReuseGraph(E.value, 0, "global", w[: E.value * E.value].view(E.value, E.value).to(_dev()))


def read_graph_file(path) -> ReuseGraph:
    return read_graph(_read(path))


def format_plan(plan: SchedulePlan) -> bytes:
    """write_plan (plan.cpp:44-69), assign/balance/read rows formatted on the GPU."""
    T = plan.node_off.shape[0]
    E = plan.order.order.numel()
    S = plan.steps_per_epoch
    has_reads = plan.read_start is not None
    return _two_call(lib().lsg_format_plan, _ptr(plan.items.contiguous()), _ptr(plan.node_off.contiguous()),
                     _ptr(plan.fetches_before.contiguous()), _ptr(plan.fetches_after.contiguous()),
                     _ptr(plan.read_start) if has_reads else None, _ptr(plan.read_end) if has_reads else None,
                     _ptr(plan.read_count) if has_reads else None, _ptr(plan.order.order.contiguous()),
                     plan.order.cost, E, T, plan.num_nodes, S, plan.dataset_size, plan.local_batch,
                     plan.chunk_threshold)


def write_plan_file(path, plan: SchedulePlan) -> None:
    _write(path, format_plan(plan))


# ---------------------------------------------------------- run reports --
# config.cpp:157-159, cost_model.hpp:13-16, pipeline.cpp:133-179: host
# formulas and the metrics.csv formatter over the device planner's and
# replay's outputs (T*N rows), byte-identical to the reference's.
@dataclass
class CostModel:
    """cost_model.hpp:13-16"""

    seek_cost: float = 13.0
    stream_cost: float = 1.0


def policy_name(policy: str) -> str:
    """config.cpp:157-159"""
    return ("clairvoyant", "lru")[_policy_code(policy)]


def _plan_costs(plan: SchedulePlan, model: CostModel, reads: bool) -> tuple[float, float]:
    """lsg_plan_costs: per-step barrier and read-plan costs summed on the
    device in the reference's order (bit-identical doubles)."""
    T, N = plan.node_off.shape[0], plan.num_nodes
    bar, io = ctypes.c_double(), ctypes.c_double()
    rs = _ptr(plan.read_start) if reads else None
    re_ = _ptr(plan.read_end) if reads else None
    rc = _ptr(plan.read_count) if reads else None
    _check(lib().lsg_plan_costs(_ptr(plan.items.contiguous()), None, _ptr(plan.node_off.contiguous()), rs, re_, rc, T,
                                N, model.seek_cost, model.stream_cost, ctypes.byref(bar), ctypes.byref(io), _stream()))
    return bar.value, io.value


def total_barrier_cost(plan: SchedulePlan, model: CostModel = CostModel()) -> float:
    """pipeline.cpp:133-138 with barrier_time (balance.cpp:41-47): the sum over
    steps of the most loaded node's fetch count x (seek + stream)."""
    return _plan_costs(plan, model, False)[0]


def total_io_cost(plan: SchedulePlan, model: CostModel = CostModel()) -> float:
    """pipeline.cpp:140-151 with read_cost (cost_model.cpp:9-18): the sum over
    steps of the slowest node's read-plan cost (seek + span x stream per
    read, in read order)."""
    if plan.read_start is None:
        raise ValidationError(3, "total_io_cost: the plan has no read plans")
    return _plan_costs(plan, model, True)[1]


def format_metrics(plan: SchedulePlan, sim: "SimResult", policy: str | None = None,
                   model: CostModel = CostModel()) -> bytes:
    """write_metrics (pipeline.cpp:153-179): one row per (epoch, step, node) in
    execution order with the replay's hits/misses, the per-node fetch counts
    before/after balancing and the step's barrier before/after."""
    per_fetch = model.seek_cost + model.stream_cost
    T, N = plan.fetches_before.shape
    S = plan.steps_per_epoch
    order = plan.order.order.cpu().numpy().view(np.uint32).tolist()
    fb = plan.fetches_before.cpu().numpy().view(np.uint32)
    fa = plan.fetches_after.cpu().numpy().view(np.uint32)
    h = sim.hits.cpu().numpy().view(np.uint32)
    m = sim.misses.cpu().numpy().view(np.uint32)
    bb = ["%.6f" % (float(v) * per_fetch) for v in fb.max(axis=1).tolist()] if N else []
    ba = ["%.6f" % (float(v) * per_fetch) for v in fa.max(axis=1).tolist()] if N else []
    pol = policy_name(policy if policy is not None else sim.policy)
    fbl, fal, hl, ml = fb.tolist(), fa.tolist(), h.tolist(), m.tolist()
    out = ["epoch,step,node,hits,misses,policy,fetches_before,fetches_after,barrier_before,barrier_after\n"]
    for g in range(T):
        head = f"{order[g // S]},{g % S},"
        tail = f",{bb[g]},{ba[g]}\n"
        out.extend(f"{head}{k},{hl[g][k]},{ml[g][k]},{pol},{fbl[g][k]},{fal[g][k]}{tail}" for k in range(N))
    return "".join(out).encode()


def write_metrics_file(path, plan: SchedulePlan, sim: "SimResult", policy: str | None = None,
                       model: CostModel = CostModel()) -> None:
    _write(path, format_metrics(plan, sim, policy, model))


def read_plan(text) -> SchedulePlan:
    """read_plan (plan.cpp:85-214) into the flat device layout. Every epoch of
    the file must have the same step count and no list more reads than
    samples (else CapabilityError: the flat layout keeps reads at item
    offsets)."""
    import numpy as np
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = ctypes.c_void_p()
    v = _lib.LsgPlanView()
    _check(lib().lsg_parse_plan(data, len(data), ctypes.byref(h), ctypes.byref(v)))
    try:
        N, T, E = v.num_nodes, v.num_steps, v.num_epochs
        arr = lambda p, n, dt: np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(dt)), shape=(n,)).copy() if n and p else np.zeros(0, np.dtype(dt))  # noqa: E731
        items = arr(v.items, v.num_items, ctypes.c_uint32)
        node_off = arr(v.node_off, T * (N + 1), ctypes.c_uint32).reshape(T, N + 1)
        fb = arr(v.fetch_before, T * N, ctypes.c_uint64).reshape(T, N)
        fa = arr(v.fetch_after, T * N, ctypes.c_uint64).reshape(T, N)
        roff = arr(v.read_off, T * N + 1, ctypes.c_uint64)
        rs = arr(v.read_start, v.num_reads, ctypes.c_uint64)
        re_ = arr(v.read_end, v.num_reads, ctypes.c_uint64)
        order = arr(v.order, E, ctypes.c_uint32)
        steps = arr(v.epoch_steps, E, ctypes.c_uint64)
        need = arr(v.needed, T * N, ctypes.c_uint64).reshape(T, N)
        red = arr(v.redundant, T * N, ctypes.c_uint64).reshape(T, N)
        meta = (v.dataset_size, v.local_batch, v.chunk_threshold, v.cost)
    finally:
        lib().lsg_free_plan(h)
    if E and (steps != steps[0]).any():
        raise CapabilityError(4, "read_plan: epochs with different step counts")
    # reads at item offsets (lsg_plan_out layout)
    gb = np.concatenate([[0], np.cumsum(node_off[:, N].astype(np.int64))])
    rstart = np.zeros(max(len(items), 1), np.uint32)
    rend = np.zeros(max(len(items), 1), np.uint32)
    rcount = (roff[1:] - roff[:-1]).reshape(T, N)
    for g in range(T):
        for k in range(N):
            n = int(rcount[g, k])
            if not n:
                continue
            if n > node_off[g, k + 1] - node_off[g, k]:
                raise CapabilityError(4, "read_plan: a list has more reads than samples")
            lo, q = int(gb[g] + node_off[g, k]), int(roff[g * N + k])
            rstart[lo:lo + n] = rs[q:q + n]
            rend[lo:lo + n] = re_[q:q + n]
    dev = _dev()
    t32 = lambda a: torch.from_numpy(np.ascontiguousarray(a).astype(np.uint32).view(np.int32)).to(dev)  # noqa: E731
    return SchedulePlan(int(meta[0]), N, int(meta[1]), int(steps[0]) if E else 0,
                        EpochOrder(t32(order), int(meta[3])), t32(items), t32(node_off), t32(fb), t32(fa),
                        t32(rstart), t32(rend), t32(rcount), t32(need), t32(red), int(meta[2]))


def read_plan_file(path) -> SchedulePlan:
    return read_plan(_read(path))


# ------------------------------------------------------------------ Store --
STORE_HEADER_BYTES = 22          # kStoreHeaderBytes (store.hpp:23)
DEFAULT_STORE_BUDGET = 1 << 30   # kDefaultStoreBudget (store.hpp:24)


@dataclass
class StoreHeader:
    """store.hpp:16-20"""
    version: int = 1
    sample_count: int = 0
    sample_size: int = 0


def create_store(path: str, sample_count: int, sample_size: int, fill_seed: int,
                 max_bytes: int = DEFAULT_STORE_BUDGET) -> None:
    """store.cpp:37-82 — SLRD file, byte-identical to the reference's; the
    splitmix64 payload is computed on the GPU."""
    _check(lib().lsg_store_create(str(path).encode(), sample_count, sample_size, fill_seed, max_bytes,
                                  _stream()))


class Store:
    """store.hpp:26-50 — read-only handle over an SLRD file (positional reads,
    safe for concurrent use). Open validates magic, version and length
    (StorageError); out-of-range reads raise ValidationError."""

    def __init__(self, path: str):
        h = ctypes.c_void_p()
        _check(lib().lsg_store_open(str(path).encode(), ctypes.byref(h)))
        self._h = h
        c, z = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().lsg_store_info(self._h, ctypes.byref(c), ctypes.byref(z)))
        self._header = StoreHeader(1, c.value, z.value)

    def header(self) -> StoreHeader:
        return self._header

    @property
    def sample_count(self) -> int:
        return self._header.sample_count

    @property
    def sample_size(self) -> int:
        return self._header.sample_size

    def read_chunk(self, start: int, count: int) -> bytes:
        """store.cpp:141-148: one contiguous read of `count` samples."""
        if count == 0:
            _check(lib().lsg_store_read(self._h, start, 0, ctypes.c_void_p(1)))
        buf = ctypes.create_string_buffer(max(1, count * self.sample_size))
        _check(lib().lsg_store_read(self._h, start, count, buf))
        return buf.raw[: count * self.sample_size]

    def read_one(self, index: int) -> bytes:
        """store.cpp:134-139"""
        return self.read_chunk(index, 1)

    def read_rows(self, ids, threshold: int = 15, out: torch.Tensor | None = None) -> torch.Tensor:
        """Samples `ids` straight into HBM rows (chunk reads of span <=
        threshold, parallel preads, one async host-to-device copy)."""
        import numpy as np
        h_ids = np.ascontiguousarray(np.asarray(ids.cpu() if isinstance(ids, torch.Tensor) else ids,
                                                dtype=np.uint32))
        n = h_ids.size
        if out is None:
            out = torch.empty((n, self.sample_size), dtype=torch.uint8, device=_dev())
        _check(lib().lsg_store_read_rows(self._h, h_ids.ctypes.data_as(ctypes.c_void_p), n, threshold,
                                         _ptr(out), _stream()))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().lsg_store_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StepFetcher:
    """The per-step loading phase for a contiguous range of ranks (lsg_fetch_step):
    owns the device arrays of buffer / batch pointers so one call fetches every
    local rank's batch of a step."""

    def __init__(self, bufs: list, outs: list, node_range: tuple[int, int], sample_bytes: int,
                 fill_seed: int, store: "Store | None" = None, threshold: int = 15):
        dev = bufs[0].device
        self.k0, self.k1 = node_range
        self.bufs, self.outs = bufs, outs
        self.pb = torch.tensor([t.data_ptr() for t in bufs], dtype=torch.int64, device=dev)
        self.po = torch.tensor([t.data_ptr() for t in outs], dtype=torch.int64, device=dev)
        self.hb = (ctypes.c_void_p * len(bufs))(*[t.data_ptr() for t in bufs])
        self.ho = (ctypes.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
        self.sample_bytes, self.fill_seed = sample_bytes, fill_seed
        self.store, self.threshold = store, threshold
        if store is not None and store.sample_size != sample_bytes:
            raise ValidationError(3, "StepFetcher: store sample size differs from sample_bytes")

    def __call__(self, items: torch.Tensor, slots: torch.Tensor, node_off_row: torch.Tensor,
                 rows_hint: int = 0) -> None:
        if self.store is not None:  # misses read from the Store file
            _check(lib().lsg_fetch_step_store(self.store._h, _ptr(self.pb), _ptr(self.po), self.hb, self.ho,
                                              _ptr(items), _ptr(slots), _ptr(node_off_row), self.k0, self.k1,
                                              rows_hint, self.threshold, _stream()))
            return
        _check(lib().lsg_fetch_step(_ptr(self.pb), _ptr(self.po), _ptr(items), _ptr(slots),
                                    _ptr(node_off_row), self.k0, self.k1, rows_hint,
                                    self.sample_bytes, self.fill_seed, _stream()))

    def fetch_steps(self, plan: "SchedulePlan", slots: torch.Tensor, host_node_off: np.ndarray,
                    step_begin: int = 0, step_end: int | None = None) -> None:
        """The loading phase of steps [step_begin, step_end) of `plan` for this
        fetcher's ranks, in step order (lsg_fetch_steps: one C call, no host
        round trips). host_node_off: the plan's [T, N+1] offsets on the host.
        Afterwards the batch tensors hold the last step's rows (rows past its
        list are unspecified)."""
        if self.store is not None:
            raise CapabilityError(4, "fetch_steps: Store-backed misses go through per-step calls")
        off = np.ascontiguousarray(host_node_off, dtype=np.uint32)
        T = off.shape[0]
        step_end = T if step_end is None else step_end
        _check(lib().lsg_fetch_steps(_ptr(self.pb), _ptr(self.po), _ptr(plan.items), _ptr(slots),
                                     _ptr(plan.node_off), ctypes.c_void_p(off.ctypes.data), step_begin, step_end,
                                     off.shape[1] - 1, self.k0, self.k1, self.sample_bytes, self.fill_seed,
                                     _stream()))


class HostRows:
    """The host tier of the miss path (lsg_host_rows): the Store payload rows
    of a dataset (store.cpp:70-80, row i at i * sample_bytes) in a tmpfs file,
    mapped and pinned so the GPU reads them over PCIe; every process of a box
    maps the same file. create=True writes it."""

    def __init__(self, path: str, count: int, sample_bytes: int, fill_seed: int = 1, create: bool = True):
        h = ctypes.c_void_p()
        _check(lib().lsg_host_rows_open(str(path).encode(), count, sample_bytes, fill_seed, int(create),
                                        ctypes.byref(h)))
        self._h, self.path, self.count, self.sample_bytes = h, str(path), count, sample_bytes

    def view(self) -> np.ndarray:
        """The rows as a [count, sample_bytes] uint8 host array (no copy)."""
        base = ctypes.c_void_p()
        _check(lib().lsg_host_rows_info(self._h, None, None, ctypes.byref(base)))
        buf = (ctypes.c_uint8 * (self.count * self.sample_bytes)).from_address(base.value)
        return np.frombuffer(buf, dtype=np.uint8).reshape(self.count, self.sample_bytes)

    def close(self) -> None:
        if self._h:
            lib().lsg_host_rows_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass


class MissStream:
    """A miss ring shared by consecutive FetchJobs of one fetch stream
    (lsg_miss_stream): each job's prefetcher runs on into the ring while the
    previous job still fetches. close() synchronises the device."""

    def __init__(self, sample_bytes: int, ring_bytes: int):
        h = ctypes.c_void_p()
        _check(lib().lsg_miss_stream_create(sample_bytes, ring_bytes, ctypes.byref(h)))
        self._h, self.sample_bytes, self.ring_bytes = h, sample_bytes, ring_bytes

    def close(self) -> None:
        if self._h:
            torch.cuda.synchronize()
            lib().lsg_miss_stream_destroy(self._h)
            self._h = None


class FetchJob:
    """The loading phase of a whole job (lsg_fetch_job): every step's batch
    for ranks node_range, hits from the HBM buffers, misses from `host` (a
    HostRows; None = the Store payload synthesised on device) into their
    batch row and new slot. The constructor builds the miss list and starts
    the miss prefetcher on `prep_stream` (which then stays busy until the
    job's misses are consumed); run() enqueues the steps on the current
    stream; stats() = {misses, kept, host_bytes, hits} (synchronous)."""

    def __init__(self, bufs: list, outs: list, node_range: tuple[int, int], plan: "SchedulePlan",
                 slots: torch.Tensor, host_node_off: np.ndarray, sample_bytes: int, fill_seed: int = 1,
                 host: HostRows | None = None, step_range: tuple[int, int] | None = None,
                 prep_stream: torch.cuda.Stream | None = None, ring_bytes: int = 0,
                 misses: MissStream | None = None):
        dev = bufs[0].device
        k0, k1 = node_range
        self._keep = [bufs, outs, plan, slots]
        self.pb = torch.tensor([t.data_ptr() for t in bufs], dtype=torch.int64, device=dev)
        self.po = torch.tensor([t.data_ptr() for t in outs], dtype=torch.int64, device=dev)
        self.off = np.ascontiguousarray(host_node_off, dtype=np.uint32)
        T = self.off.shape[0]
        g0, g1 = step_range if step_range is not None else (0, T)
        d = _lib.LsgFetchJobDesc()
        d.d_bufs, d.d_outs = self.pb.data_ptr(), self.po.data_ptr()
        d.d_items, d.d_slots, d.d_node_off = plan.items.data_ptr(), slots.data_ptr(), plan.node_off.data_ptr()
        d.h_node_off = self.off.ctypes.data
        d.step_begin, d.step_end, d.N = g0, g1, self.off.shape[1] - 1
        d.node_begin, d.node_end = k0, k1
        d.sample_bytes, d.fill_seed = sample_bytes, fill_seed
        d.host = host._h if host is not None else None
        d.ring_bytes = ring_bytes
        d.misses = misses._h if misses is not None else None
        self.host, self.misses = host, misses
        if prep_stream is None:  # with a host tier the prefetcher holds its stream: never the fetch's
            prep_stream = torch.cuda.Stream(device=dev) if host is not None else torch.cuda.current_stream()
        st = prep_stream
        if host is not None:
            st.wait_stream(torch.cuda.current_stream())  # the plan and the replay's slots
        self._prep = st
        h = ctypes.c_void_p()
        _check(lib().lsg_fetch_job_create(ctypes.byref(d), ctypes.byref(h), ctypes.c_void_p(st.cuda_stream)))
        self._h = h

    def run(self) -> None:
        _check(lib().lsg_fetch_job_run(self._h, _stream()))

    def stats(self) -> dict:
        a = (ctypes.c_uint64 * 4)()
        _check(lib().lsg_fetch_job_stats(self._h, a, _stream()))
        return {"misses": a[0], "kept": a[1], "host_bytes": a[2], "hits": a[3]}

    def close(self, stream: torch.cuda.Stream | None = None) -> None:
        """Free the job's device state, stream-ordered after its work on
        `stream` (default: the current stream, where run() enqueued it)."""
        if self._h:
            st = stream if stream is not None else torch.cuda.current_stream()
            lib().lsg_fetch_job_destroy(self._h, ctypes.c_void_p(st.cuda_stream))
            for t in (self.pb, self.po):
                t.record_stream(st)
            self._h = None

