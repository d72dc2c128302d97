"""Per-stage device timings (CUDA events) of the planner, repeated."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00224_b200 as ls  # noqa: E402
from time_plan import CFGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
D, E, N, b, C = CFGS[name]
tc = ls.TraceConfig(D, E, N, b, 42, True)
pc = ls.PipelineConfig(trace=tc, buffer_capacity=C)
for r in range(reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    tr = ls.generate_trace(tc)
    ev[1].record()
    g = ls.build_reuse_graph(tr, C)
    ev[2].record()
    p = ls.pso_order(g, pc.pso)
    ev[3].record()
    out = ls.plan_schedule(pc)
    ev[4].record()
    torch.cuda.synchronize()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
    print(f"{name} rep {r}: trace {t[0]:.2f} ms  graph {t[1]:.2f}  pso {t[2]:.2f}  plan_schedule {t[3]:.2f}")
