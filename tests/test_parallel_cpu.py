"""World-size-2 gloo tests of the multi-GPU host logic on CPU: rank ranges
partition the training ranks, the all-gather of per-GPU replay columns
reproduces the reference replay rows (oracle), and the all-gather of reuse
matrix row blocks reproduces the whole matrix (oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2211_00224_b200.parallel import allgather_blocks, combine_rows, rank_range


def test_rank_range_partitions():
    for N in (1, 3, 8, 32, 256):
        for world in (1, 2, 3, 4, 8):
            if world > N:
                continue
            spans = [rank_range(N, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(k1 - k0 for k0, k1 in spans) - min(k1 - k0 for k0, k1 in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = O.Cfg(600, 4, 5, 6, seed=3, buffer_capacity=70, pso_iters=20)
        p = O.plan(c)
        h, m = O.simulate(p.items, p.node_off, 5, 600, 70)
        k0, k1 = rank_range(5, world, rank)
        # what this GPU's replay produces: only its own columns
        hl = torch.zeros(h.shape, dtype=torch.int64)
        ml = torch.zeros(m.shape, dtype=torch.int64)
        hl[:, k0:k1] = torch.from_numpy(h[:, k0:k1].astype(np.int64))
        ml[:, k0:k1] = torch.from_numpy(m[:, k0:k1].astype(np.int64))
        combine_rows(hl, ml)
        ok = bool(np.array_equal(hl.numpy(), h)) and bool(np.array_equal(ml.numpy(), m))
        # reuse-matrix row blocks (uneven split: E=7 over the world)
        tr = O.generate_trace(900, 7, 3, 10, 5, True)
        w = O.build_reuse_graph(tr, 900, 3, 10, 100, "pernode", True).astype(np.int64)
        u0, u1 = rank_range(7, world, rank)
        full = allgather_blocks(torch.from_numpy(w[u0:u1].copy()), 7)
        ok = ok and bool(np.array_equal(full.numpy(), w))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_replay_rows_combine_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    assert all(ok for _, ok in res), res
