"""Where does a replay launched beside a running plan wait? Host timings of
the lsg_simulate call and of the stream sync, with a plan on another stream."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_00224_b200 as ls
from paper_2211_00224_b200.loadsched import _ptr

D, E, N, b, C = 262144, 100, 8, 512, 52428
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
plan = ls.plan_schedule(pc).plan
T = plan.node_off.shape[0]
hits = torch.zeros((T, N), dtype=torch.int32, device="cuda")
misses = torch.zeros_like(hits)
slots = torch.empty(plan.items.numel(), dtype=torch.int32, device="cuda")
R, P = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=-1)

def sim():
    t0 = time.perf_counter()
    rc = ls.lib().lsg_simulate(_ptr(plan.items), _ptr(plan.node_off), T, N, D, C, 0, 0, N, _ptr(hits), _ptr(misses),
                              _ptr(slots), __import__("ctypes").c_void_p(R.cuda_stream))
    t1 = time.perf_counter()
    R.synchronize()
    t2 = time.perf_counter()
    return rc, round(1e3 * (t1 - t0), 1), round(1e3 * (t2 - t1), 1)

for _ in range(2):
    sim()
print("alone", sim(), flush=True)
for it in range(3):
    def planner():
        torch.cuda.set_device(0)
        with torch.cuda.stream(P):
            t0 = time.perf_counter()
            ls.plan_schedule(pc)
            print("  plan host", round(1e3 * (time.perf_counter() - t0), 1), flush=True)
    th = threading.Thread(target=planner)
    th.start()
    time.sleep(0.05)
    print("beside plan", it, sim(), flush=True)
    th.join()
    torch.cuda.synchronize()
