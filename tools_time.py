import time, json, torch, sys
sys.path.insert(0, '.')
import paper_2211_00224_b200 as ls
def ev(): return torch.cuda.Event(enable_timing=True)
def timeit(f, reps=2):
    f(); torch.cuda.synchronize()
    ts=[]
    for _ in range(reps):
        a,b=ev(),ev(); a.record(); r=f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts), r
for name,(D,E,N,b,C,mode) in {"cfg1":(16384,10,4,64,1638,"global"),"cfg2":(262144,100,8,512,52428,"global"),
                         "cfg2pn":(262144,100,8,512,52428,"pernode"),"cfg4":(131072,500,8,64,6553,"global")}.items():
    tc=ls.TraceConfig(D,E,N,b,42,True)
    pc=ls.PipelineConfig(trace=tc,buffer_capacity=C,graph_mode=mode)
    t_tr, tr = timeit(lambda: ls.generate_trace(tc))
    t_g, g = timeit(lambda: ls.build_reuse_graph(tr, C, mode))
    p=ls.PsoParams(seed=42)
    t_p, pr = timeit(lambda: ls.pso_order(g, p), 1)
    if name=="cfg4":
        print(json.dumps(dict(cfg=name, trace_ms=t_tr, graph_ms=t_g, pso_ms=t_p, pso_iters=pr.iterations)), flush=True); continue
    t_plan, out = timeit(lambda: ls.plan_schedule(pc), 1)
    t_sim, sim = timeit(lambda: ls.simulate_plan(out.plan, C), 1)
    A = E*tc.keep()
    print(json.dumps(dict(cfg=name, trace_ms=t_tr, graph_ms=t_g, pso_ms=t_p, pso_iters=pr.iterations, plan_ms=t_plan, sim_ms=t_sim,
          plan_Msps=A/t_plan/1e3, misses=sim.total_misses, hits=sim.total_hits)), flush=True)
