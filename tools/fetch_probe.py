"""Fetch phase alone for r local ranks (the per-GPU share at 8/r GPUs):
wall time of lsg_fetch_steps over the whole cfg2 job vs its algorithmic
bytes, to expose per-step overheads."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2211_00224_b200 as ls

D, E, N, b, C, SB = 262144, 100, 8, 512, 52428, 262144
if os.environ.get("PROBE_CFG") == "cfg3":  # 16 MiB samples, 128 GiB buffer per rank
    D, E, N, b, C, SB = 65536, 10, 8, 8, 8192, 16 << 20
pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, 42, True), buffer_capacity=C)
plan = ls.plan_schedule(pc).plan
res = {}
for r in [int(x) for x in (sys.argv[1:] or ["1", "2", "8"])]:
    bufs = [torch.empty((C, SB), dtype=torch.uint8, device="cuda") for _ in range(r)]
    outs = [torch.empty((2 * b, SB), dtype=torch.uint8, device="cuda") for _ in range(r)]
    f = ls.StepFetcher(bufs, outs, (0, r), SB, 1)
    sim = ls.simulate_plan(plan, C, node_range=(0, r), want_slots=True)
    off = plan.node_off.cpu().numpy()
    hits = int(sim.hits[:, :r].sum()); miss = int(sim.misses[:, :r].sum())
    for _ in range(2):
        f.fetch_steps(plan, sim.slots, off)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); f.fetch_steps(plan, sim.slots, off); z.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(z)
    # the job's kernels alone (creation -- miss list, row flags -- outside the events)
    j = ls.FetchJob(bufs, outs, (0, r), plan, sim.slots, off, SB, 1)
    torch.cuda.synchronize()
    a.record(); j.run(); z.record(); torch.cuda.synchronize()
    run_ms = a.elapsed_time(z)
    j.close()
    alg = 2 * SB * hits + 2 * SB * miss
    res[r] = {"fetch_ms": round(ms, 1), "TBps": round(alg / ms / 1e9, 3), "us_per_step": round(ms * 1e3 / off.shape[0], 1),
              "run_ms": round(run_ms, 1), "run_TBps": round(alg / run_ms / 1e9, 3),
              "run_us_per_step": round(run_ms * 1e3 / off.shape[0], 1),
              "data_us_per_step_at_6.55": round(alg / 6.55e12 * 1e6 / off.shape[0], 1)}
    del bufs, outs, f, sim
    torch.cuda.empty_cache()
print(json.dumps(res))
