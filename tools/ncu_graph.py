"""Driver for ncu captures of K1 (shuffle) and K2/K3 (reuse matrix):
cfg2 trace (D=262144, E=100) and the cfg4 reuse matrix (D=131072, E=500,
N=8, b=64, C=6553; Global and PerNode). Prints CUDA-event timings when run
without ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00224_b200 as ls  # noqa: E402

ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
t2 = ls.TraceConfig(262144, 100, 8, 512, 42, True)
t4 = ls.TraceConfig(131072, 500, 8, 64, 42, True)
for rep in range(2):
    e = [ev() for _ in range(5)]
    e[0].record()
    tr2 = ls.generate_trace(t2)
    e[1].record()
    tr4 = ls.generate_trace(t4)
    e[2].record()
    g = ls.build_reuse_graph(tr4, 6553, "global")
    e[3].record()
    gp = ls.build_reuse_graph(tr4, 6553, "pernode")
    e[4].record()
    torch.cuda.synchronize()
    t = [e[i].elapsed_time(e[i + 1]) for i in range(4)]
    print(f"rep {rep}: cfg2 trace {t[0]:.3f} ms  cfg4 trace {t[1]:.3f} ms  cfg4 graph global {t[2]:.3f} ms  "
          f"pernode {t[3]:.3f} ms  (w sum {int(g.weights.sum())}, {int(gp.weights.sum())})", flush=True)
