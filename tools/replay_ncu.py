"""One replay (simulate_plan with slots) of a cfg5 shape for an ncu capture of
k_replay_chain: python tools/replay_ncu.py N E"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_00224_b200 as ls  # noqa: E402

N, E = int(sys.argv[1]), int(sys.argv[2])
D, b = 1 << 20, 512
C = D // (2 * N)
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
plan = ls.plan_schedule(pc).plan
sim = ls.simulate_plan(plan, C, want_slots=len(sys.argv) > 3)
torch.cuda.synchronize()
print(N, E, sim.total_hits, sim.total_misses, plan.items.numel())
