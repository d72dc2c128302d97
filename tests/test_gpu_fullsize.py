"""Full-size parity: the CUDA path at the BASELINE.json shapes vs digests of
the UNMODIFIED reference's own outputs at the same shapes.

tests/golden/full_shapes.json holds SHA-256 digests (and the small outputs
inline) of plan_schedule (pipeline.cpp:32-120) + simulate_plan
(buffer.cpp:183-247) run by oracle/_ref/ref_dump on cfg1, cfg2 (Global and
PerNode, E=100), cfg4 (E=500) and cfg5 (E=3 at 32 and 256 logical ranks);
tools/make_goldens.py made them. Here the same configs run through the
sm_100a path and every output array is hashed in the same layout: trace,
reuse graph, epoch order, PSO history and iteration count, node lists
(ids + hit tags), node offsets, fetch counts before/after balancing, chunk
reads, and the replay's per-(step, node) hits/misses. Bit-exact or failed.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_shapes.json")))
NAMES = [k for k in GOLD if not k.startswith("_")]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def u32(t):
    return t.detach().cpu().numpy().view(np.uint32)


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def pc_of(ls, c: dict):
    return ls.PipelineConfig(
        trace=ls.TraceConfig(c["dataset_size"], c["num_epochs"], c["num_nodes"], c["local_batch"], c["seed"], True),
        buffer_capacity=c["buffer_capacity"], graph_mode=c.get("graph_mode", "global"))


@pytest.mark.parametrize("name", NAMES)
def test_full_shape_matches_reference(ls, name):
    g = GOLD[name]
    c = g["config"]
    N = c["num_nodes"]
    out = ls.plan_schedule(pc_of(ls, c))
    p = out.plan
    sim = ls.simulate_plan(p, c["buffer_capacity"])
    arrays = {
        "trace": u32(out.trace.epochs), "graph": u64(out.graph.weights), "items": u32(p.items),
        "nodeoff": u32(p.node_off), "fb": u32(p.fetches_before), "fa": u32(p.fetches_after),
        "hits": u32(sim.hits), "misses": u32(sim.misses), "rcount": u32(p.read_count),
        "rneed": u32(p.read_needed), "rred": u32(p.read_redundant),
        "reads": O.compact_reads(u32(p.read_start), u32(p.read_end), u32(p.read_count), u32(p.node_off), N),
    }
    bad = [k for k, a in arrays.items() if (a.size, sha(a)) != (g["arrays"][k]["n"], g["arrays"][k]["sha256"])]
    assert not bad, f"{name}: arrays differing from the reference: {bad}"
    assert u32(p.order.order).tolist() == g["order"] and p.order.cost == g["cost"]
    assert (sim.total_hits, sim.total_misses) == (g["total_hits"], g["total_misses"])
    if "history" in g:
        assert out.pso is not None
        assert out.pso.iterations == g["iterations"]
        assert u64(out.pso.history).tolist() == g["history"]
