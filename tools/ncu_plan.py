import sys, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2211_00224_b200 as ls
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4
pc = ls.PipelineConfig(trace=ls.TraceConfig(262144, E, 8, 512, 42, True), buffer_capacity=52428)
out = ls.plan_schedule(pc)
torch.cuda.synchronize()
print("ok", int(out.plan.node_off[-1, -1]))
