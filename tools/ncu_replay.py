"""Plan a cfg5-shaped job, then replay it (ncu target: k_replay_cta)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00224_b200 as ls  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 32
E = int(sys.argv[2]) if len(sys.argv) > 2 else 3
D = 1 << 20
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, 512, 42, True), buffer_capacity=D // (2 * N))
out = ls.plan_schedule(pc)
torch.cuda.synchronize()
sim = ls.simulate_plan(out.plan, D // (2 * N))
torch.cuda.synchronize()
print("ok", sim.total_hits, sim.total_misses)
