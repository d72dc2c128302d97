"""K7 replay timing: simulate_plan (next-use pass + forward replay) at cfg2
(8 ranks) and a cfg5 shape, segmented vs serial next-use pass."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_00224_b200 as ls  # noqa: E402

ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {}
shapes = {"cfg2": (262144, 100, 8, 512, 52428), "cfg5_n32_e10": (1 << 20, 10, 32, 512, 16384),
          "cfg5_n256_e10": (1 << 20, 10, 256, 512, 2048)}
for name, (D, E, N, b, C) in shapes.items():
    if len(sys.argv) > 1 and name not in sys.argv[1:]:
        continue
    pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
    plan = ls.plan_schedule(pc).plan
    out = {}
    for mode in ("segmented", "serial"):
        if mode == "serial":
            os.environ["LSG_NEXTUSE_SERIAL"] = "1"
        ts = []
        for _ in range(3):
            a, z = ev(), ev()
            a.record()
            sim = ls.simulate_plan(plan, C, want_slots=True)
            z.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(z))
        os.environ.pop("LSG_NEXTUSE_SERIAL", None)
        out[mode] = {"ms": [round(t, 2) for t in ts], "hits": sim.total_hits, "misses": sim.total_misses}
    res[name] = out
print(json.dumps(res))
