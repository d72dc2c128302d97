"""Multi-GPU timings of the other BASELINE shapes (torchrun, one process per
GPU, NCCL): cfg4's 500x500 reuse matrix with row-sharded K3 + all-gather, and
cfg5's replay (1M ids, N simulated ranks) sharded by rank + all-gather of the
rows. Device time, max over ranks; one JSON line from rank 0."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2211_00224_b200 as ls
from paper_2211_00224_b200.parallel import sharded_reuse_graph, sharded_simulate


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        z.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(z)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        best = float(t) if best is None else min(best, float(t))
    return best


local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
res = {"world": world}
t4 = ls.generate_trace(ls.TraceConfig(131072, 500, 8, 64, 42, True))
for mode in ("global", "pernode"):
    res[f"cfg4_graph_{mode}_ms"] = timed(lambda: sharded_reuse_graph(ls, t4, 6553, mode))
for n_ranks, E in ((256, 10), (32, 10)):
    C = (1 << 20) // (2 * n_ranks)
    pc = ls.PipelineConfig(trace=ls.TraceConfig(1 << 20, E, n_ranks, 512, 42, True), buffer_capacity=C)
    plan = ls.plan_schedule(pc).plan
    res[f"cfg5_N{n_ranks}_E{E}_replay_ms"] = timed(lambda: sharded_simulate(ls, plan, C, world, rank))
if rank == 0:
    print(json.dumps(res), flush=True)
dist.destroy_process_group()
