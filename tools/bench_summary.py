import json,sys
for line in sys.stdin:
    if not line.startswith('{"metric"'): continue
    d=json.loads(line)
    print({k:round(d[k],1) for k in ("value","ms_per_step","plan_ms","replay_ms","fetch_ms","single_job_ms")}, "frac", round(d["roofline"]["frac"],3), "e2e", round(d.get("e2e",{}).get("value",0)), d["config"]["parallelism"], "launches", d["gpu_launches"])
