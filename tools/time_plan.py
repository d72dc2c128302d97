"""Planner timing across the BASELINE config shapes (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_00224_b200 as ls  # noqa: E402

CFGS = {
    "cfg1": (16384, 10, 4, 64, 1638),
    "cfg2": (262144, 100, 8, 512, 52428),
    "cfg3": (65536, 10, 8, 8, 8192),
    "cfg4": (131072, 500, 8, 64, 6553),
    "cfg5_N32_E3": (1 << 20, 3, 32, 512, (1 << 20) // 64),
    "cfg5_N32_E10": (1 << 20, 10, 32, 512, (1 << 20) // 64),
    "cfg5_N64_E10": (1 << 20, 10, 64, 512, (1 << 20) // 128),
    "cfg5_N128_E10": (1 << 20, 10, 128, 512, (1 << 20) // 256),
    "cfg5_N256_E10": (1 << 20, 10, 256, 512, (1 << 20) // 512),
    # full cfg5 (BASELINE configs[4]: 1,000 epochs)
    "cfg5_N32_E1000": (1 << 20, 1000, 32, 512, (1 << 20) // 64),
    "cfg5_N64_E1000": (1 << 20, 1000, 64, 512, (1 << 20) // 128),
    "cfg5_N128_E1000": (1 << 20, 1000, 128, 512, (1 << 20) // 256),
    "cfg5_N256_E1000": (1 << 20, 1000, 256, 512, (1 << 20) // 512),
}
if __name__ != "__main__":
    names = []
else:
    names = sys.argv[1:] or list(CFGS)
for name in names:
    D, E, N, b, C = CFGS[name]
    pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
    out = ls.plan_schedule(pc)
    ls.simulate_plan(out.plan, C)  # warm the pool / modules for both phases
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    out = ls.plan_schedule(pc)
    ev[1].record()
    sim = ls.simulate_plan(out.plan, C)
    ev[2].record()
    torch.cuda.synchronize()
    A = E * pc.trace.keep()
    pm, sm = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    print(f"{name:14s} plan {pm:9.1f} ms ({A / pm / 1e3:7.2f} M samples/s, {pm * 1e3 / (E * pc.trace.steps_per_epoch()):7.1f} us/step)"
          f"  replay {sm:8.1f} ms  misses {sim.total_misses} hits {sim.total_hits}", flush=True)
