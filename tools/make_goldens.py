#!/usr/bin/env python
"""tools/make_goldens.py — TEST INFRASTRUCTURE: full-size reference goldens.

Runs the UNMODIFIED reference (oracle/_ref/ref_dump, compiled from
/root/reference/proj/src by oracle/Makefile) on the BASELINE.json shapes at
their full size — plan_schedule (pipeline.cpp:32-120) + simulate_plan
(buffer.cpp:183-247) — and writes SHA-256 digests of every output array into
tests/golden/full_shapes.json. The -m gpu test tests/test_gpu_fullsize.py
hashes the device arrays of the same configs and compares. Small outputs
(order, cost, PSO history, iteration count, totals) are stored inline.

Arrays are hashed in the layout the CUDA path emits (ref_dump.cpp dump_plan):
  trace   u32 [E][keep]          graph  u64 [E][E]
  items   u32 id | hit<<31       nodeoff u32 [T][N+1]   fb/fa u32 [T][N]
  hits/misses u32 [T][N]         reads: rcount/rneed/rred u32 [T][N] and the
  valid read spans (rstart, rend) of every list concatenated (u32 pairs).

Run here (needs /root/reference at build time); cfg4 takes ~10 min of one
core, the whole set ~15 min with one process per config:
    python tools/make_goldens.py [name ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
from oracle import compact_reads  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
OUT = os.path.join(ROOT, "tests", "golden", "full_shapes.json")

# name -> reference config keys (config.cpp:63-97); seed 42, drop_last=1 and the
# PipelineConfig defaults (config.hpp:17-36) unless given. Shapes: SURVEY.md §8d.
CONFIGS = {
    "cfg1": dict(dataset_size=16384, num_epochs=10, num_nodes=4, local_batch=64, buffer_capacity=1638),
    "cfg2_global": dict(dataset_size=262144, num_epochs=100, num_nodes=8, local_batch=512,
                        buffer_capacity=52428),
    "cfg2_pernode": dict(dataset_size=262144, num_epochs=100, num_nodes=8, local_batch=512,
                         buffer_capacity=52428, graph_mode="pernode"),
    "cfg4": dict(dataset_size=131072, num_epochs=500, num_nodes=8, local_batch=64, buffer_capacity=6553),
    "cfg5_n32": dict(dataset_size=1048576, num_epochs=3, num_nodes=32, local_batch=512,
                     buffer_capacity=16384),
    "cfg5_n256": dict(dataset_size=1048576, num_epochs=3, num_nodes=256, local_batch=512,
                      buffer_capacity=2048),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def digest_dir(d: str, cfg: dict) -> dict:
    N = cfg["num_nodes"]
    rd = lambda n, t: np.fromfile(os.path.join(d, n), dtype=t)  # noqa: E731
    out = {}
    for name, t in (("trace", np.uint32), ("graph", np.uint64), ("items", np.uint32),
                    ("nodeoff", np.uint32), ("fb", np.uint32), ("fa", np.uint32),
                    ("hits", np.uint32), ("misses", np.uint32), ("rcount", np.uint32),
                    ("rneed", np.uint32), ("rred", np.uint32)):
        a = rd(f"{name}.{'u64' if t == np.uint64 else 'u32'}", t)
        out[name] = {"sha256": sha(a), "n": int(a.size)}
    reads = compact_reads(rd("rstart.u32", np.uint32), rd("rend.u32", np.uint32), rd("rcount.u32", np.uint32),
                          rd("nodeoff.u32", np.uint32), N)
    out["reads"] = {"sha256": sha(reads), "n": int(reads.size)}
    g = rd("graph.u64", np.uint64)
    hits, misses = rd("hits.u32", np.uint32), rd("misses.u32", np.uint32)
    small = {
        "order": rd("order.u32", np.uint32).tolist(),
        "cost": int(rd("cost.u64", np.uint64)[0]),
        "graph_sum": int(g.sum(dtype=np.uint64)),
        "total_hits": int(hits.sum(dtype=np.uint64)),
        "total_misses": int(misses.sum(dtype=np.uint64)),
    }
    if os.path.exists(os.path.join(d, "hist.u64")):
        small["history"] = rd("hist.u64", np.uint64).tolist()
        small["iterations"] = int(rd("iters.u32", np.uint32)[0])
    return {"arrays": out, **small}


def run_one(name: str) -> tuple[str, dict]:
    cfg = CONFIGS[name]
    kv = [f"seed=42"] + [f"{k}={v}" for k, v in cfg.items()]
    with tempfile.TemporaryDirectory(dir="/tmp") as d:
        t0 = time.time()
        env = dict(os.environ, REF_DUMP_NO_RESIDENCY="1")
        subprocess.run([REF_DUMP, "plan", d, *kv], check=True, env=env)
        el = time.time() - t0
        res = digest_dir(d, cfg)
    res["config"] = {"seed": 42, **cfg}
    res["reference_seconds_plan_and_simulate"] = round(el, 1)
    print(f"{name}: {el:.1f} s  hits={res['total_hits']} misses={res['total_misses']} cost={res['cost']}",
          flush=True)
    return name, res


def main():
    names = sys.argv[1:] or list(CONFIGS)
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    data.setdefault("_about", "SHA-256 of the UNMODIFIED reference's outputs (oracle/_ref/ref_dump plan, "
                    "plan_schedule + simulate_plan) at full BASELINE shapes; made by tools/make_goldens.py")
    with ThreadPoolExecutor(len(names)) as ex:
        for name, res in ex.map(run_one, names):
            data[name] = res
            os.makedirs(os.path.dirname(OUT), exist_ok=True)
            json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
