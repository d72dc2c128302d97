"""Replay (K7, r ranks) alone vs beside a full-job fetch on another stream."""
import json, os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_00224_b200 as ls

r = int(sys.argv[1]) if len(sys.argv) > 1 else 8
D, E, N, b, C, SB = 262144, 100, 8, 512, 52428, 262144
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
plan = ls.plan_schedule(pc).plan
bufs = [torch.empty((C, SB), dtype=torch.uint8, device="cuda") for _ in range(8)]
outs = [torch.empty((1024, SB), dtype=torch.uint8, device="cuda") for _ in range(8)]
f = ls.StepFetcher(bufs, outs, (0, 8), SB, 1)
sim8 = ls.simulate_plan(plan, C, want_slots=True)
off = plan.node_off.cpu().numpy()
F = torch.cuda.Stream()
ev = lambda: torch.cuda.Event(enable_timing=True)

def replay():
    a, z = ev(), ev()
    a.record(); ls.simulate_plan(plan, C, node_range=(0, r), want_slots=True); z.record()
    torch.cuda.synchronize()
    return a.elapsed_time(z)

def plan1():
    a, z = ev(), ev()
    a.record(); ls.plan_schedule(pc); z.record()
    torch.cuda.synchronize()
    return a.elapsed_time(z)

res = {"alone_replay": [replay() for _ in range(3)], "alone_plan": [plan1() for _ in range(2)]}
P = torch.cuda.Stream()
out = []
for _ in range(2):
    def planner():
        torch.cuda.set_device(0)
        with torch.cuda.stream(P):
            ls.plan_schedule(pc)
    th = threading.Thread(target=planner)
    th.start()
    import time; time.sleep(0.03)
    out.append(replay())
    th.join(); torch.cuda.synchronize()
res["beside_plan_replay"] = out
for what, fn in (("replay", replay), ("plan", plan1)):
    out = []
    for _ in range(2):
        def fetch():
            torch.cuda.set_device(0)
            with torch.cuda.stream(F):
                f.fetch_steps(plan, sim8.slots, off, 0, 2000)
        th = threading.Thread(target=fetch)
        th.start()
        import time; time.sleep(0.05)
        out.append(fn())
        th.join(); torch.cuda.synchronize()
    res["beside_fetch_" + what] = out
print(json.dumps({k: [round(x, 1) for x in v] for k, v in res.items()}))
