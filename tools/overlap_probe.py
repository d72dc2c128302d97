"""Probe: does the 1-CTA plan loop overlap with the fetch phase on one GPU?
Times plan alone, fetch alone, and both concurrently (plan on its own stream
from a worker thread; the fetch loop on another stream)."""
import sys, os, threading, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_00224_b200 as ls

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 8
D, E, N, b, C, SB = 262144, 100, 8, 512, 52428, 262144
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
dev = torch.device("cuda", 0)
k0, k1 = 0, nr
bufs = [torch.empty((C, SB), dtype=torch.uint8, device=dev) for _ in range(k0, k1)]
outs = [torch.empty((1024, SB), dtype=torch.uint8, device=dev) for _ in range(k0, k1)]
fetcher = ls.StepFetcher(bufs, outs, (k0, k1), SB, 1)
out = ls.plan_schedule(pc)
plan = out.plan
sim = ls.simulate_plan(plan, C, node_range=(k0, k1), want_slots=True)
off = plan.node_off.cpu().numpy()
T = off.shape[0]
bases = [0]
for g in range(T):
    bases.append(bases[-1] + int(off[g, N]))

def fetch_all():
    items, slots, noff = plan.items, sim.slots, plan.node_off
    for g in range(T):
        fetcher(items[bases[g]:], slots[bases[g]:], noff[g], int(off[g, k1]) - int(off[g, k0]))

P, F = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn, stream):
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(); fn(); z.record()
    return a, z

for _ in range(2):
    fetch_all(); ls.plan_schedule(pc)
torch.cuda.synchronize()
res = {}
a, z = timed(lambda: ls.plan_schedule(pc), P); torch.cuda.synchronize(); res["plan_alone_ms"] = a.elapsed_time(z)
t0 = time.time(); a, z = timed(fetch_all, F); torch.cuda.synchronize(); res["fetch_alone_ms"] = a.elapsed_time(z); res["fetch_alone_wall"] = (time.time()-t0)*1e3
for rep in range(2):
    box = {}
    def worker():
        box["ev"] = timed(lambda: ls.plan_schedule(pc), P)
    th = threading.Thread(target=worker)
    t0 = time.time()
    th.start()
    a2, z2 = timed(fetch_all, F)
    th.join(); torch.cuda.synchronize()
    res[f"conc{rep}_wall_ms"] = (time.time() - t0) * 1e3
    res[f"conc{rep}_plan_ms"] = box["ev"][0].elapsed_time(box["ev"][1])
    res[f"conc{rep}_fetch_ms"] = a2.elapsed_time(z2)
print(json.dumps(res))
