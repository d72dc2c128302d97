import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2211_00224_b200 as ls
for E in (20, 100):
    pc = ls.PipelineConfig(trace=ls.TraceConfig(262144, E, 8, 512, 42, True), buffer_capacity=52428)
    ls.plan_schedule(pc); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ls.plan_schedule(pc); b.record(); torch.cuda.synchronize()
    print("E", E, "plan ms", a.elapsed_time(b), flush=True)
