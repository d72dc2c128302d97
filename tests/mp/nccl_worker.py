"""torchrun worker for tests/test_gpu_multi.py (one process per GPU, NCCL).

Checks, on every rank, that the sharded multi-GPU path equals the
single-GPU one bit for bit: the row-sharded reuse matrix (all-gather of row
blocks) and the rank-sharded replay (all-gather of per-rank hit/miss
columns). Prints one JSON line per rank."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2211_00224_b200 as ls  # noqa: E402
from paper_2211_00224_b200.parallel import sharded_reuse_graph, sharded_simulate  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = {}
    # K3 rows: cfg4 shape (E=500) and a PerNode case
    for name, tc, C, mode in (("cfg4", ls.TraceConfig(131072, 500, 8, 64, 42, True), 6553, "global"),
                              ("pernode", ls.TraceConfig(20000, 37, 5, 16, 3, False), 900, "pernode")):
        t = ls.generate_trace(tc)
        want = ls.build_reuse_graph(t, C, mode).weights
        got = sharded_reuse_graph(ls, t, C, mode).weights
        ok[name] = bool(torch.equal(got, want))
    # K7: rank-sharded replay rows vs the whole replay
    pc = ls.PipelineConfig(trace=ls.TraceConfig(16384, 6, 8, 64, 42, True), buffer_capacity=1638)
    plan = ls.plan_schedule(pc).plan
    full = ls.simulate_plan(plan, 1638)
    sim, _ = sharded_simulate(ls, plan, 1638, world, rank)
    ok["replay"] = bool(torch.equal(sim.hits, full.hits)) and bool(torch.equal(sim.misses, full.misses)) \
        and sim.total_hits == int(full.hits.sum()) and sim.total_misses == int(full.misses.sum())
    line = json.dumps({"rank": rank, "world": world, "ok": ok})
    out_dir = os.environ.get("LSG_MP_OUT")
    if out_dir:  # one file per rank (stdout lines of the ranks can interleave)
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            f.write(line)
    else:
        print(line, flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0 if all(ok.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
