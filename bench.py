#!/usr/bin/env python
"""bench.py — the SOLAR loading path on B200 (driver contract: one JSON line).

One bench *step* is one full pass of the hot path over one job. The default
job is cfg2 (BASELINE.json configs[1]: 262,144 PtychoNN-shaped samples of
256x256 fp32, 100 epochs, 8 ranks, local batch 512, per-rank HBM buffer 20%
of the dataset); `--config cfg1|cfg3|cfg4|cfg5` runs the other named shapes
(cfg4/cfg5: plan + replay only, as BASELINE names them):

  plan     K1 shuffle -> K2/K3 reuse matrix -> K4 PSO order -> K5/K6 step loop
           (locality remap, balance, clairvoyant eviction)   [one GPU per job:
           job i on GPU i mod N, node lists broadcast over NVLink (NCCL)]
  replay   K7 per-rank Belady replay of this GPU's ranks + NCCL all-gather of
           the per-(step, rank) hit/miss rows                [sharded by rank]
  fetch    every training step's batch of this GPU's ranks through the fused
           TMA step kernel: hits from the rank's 12.8 GiB HBM sample buffer,
           misses written into the batch and their slot — in `value` from the
           Store payload computed on device, in `e2e` read over PCIe from the
           host tier (the dataset's payload rows pinned in host memory)

Jobs are pipelined: plans run on their own stream (the step loop is ONE
persistent CTA) from a helper thread, overlapping earlier jobs' replay and
fetch on the other SMs. `single_job_ms` is one job alone, unpipelined.

value = planned-and-fetched samples of the K timed jobs / timed region (max
over ranks). `e2e` = the same through the host-buffer API (plan to pinned
host and back, hit/miss rows read back, every miss over PCIe). The roofline
object is the fetch phase (HBM-bound gather; hit bytes only);
`verify` is a one-shot byte check of the benched fetch (off the timed region).

--impl reference times the reference's own CPU implementation (oracle/_ref,
compiled from /root/reference/proj/src): plan_schedule + simulate_plan of the
FULL job on one core (cfg5: E = 1 and 3, linear in E) plus Store::read_one
batch fetches on every host core.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# more hardware work queues than the default 8, so the plan / replay / fetch
# streams never share one (a shared queue serialises a replay behind the
# planner's persistent kernel); must be set before CUDA initialises
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "plan samples/s (shuffle+order+evict+assign); HBM-buffer gather GB/s; 1-8 GPU"
# BASELINE.json configs; b, E and C where BASELINE leaves them open are
# SURVEY.md §8d's choices. kind "job" = plan + replay + batch fetch of the
# whole job; "plan" = plan + replay (cfg4: reuse matrix + ordering stress,
# cfg5: replay + assignment sweep over logical ranks).
CONFIGS = {
    "cfg1": dict(D=16384, E=10, N=4, b=64, C=1638, sample_bytes=256 * 256 * 4, kind="job",
                 label="PtychoNN-shaped, 10%/rank"),
    "cfg2": dict(D=262144, E=100, N=8, b=512, C=52428, sample_bytes=256 * 256 * 4, kind="job",
                 label="PtychoNN-shaped, 20%/rank"),
    "cfg3": dict(D=65536, E=10, N=8, b=8, C=8192, sample_bytes=4 * 128 ** 3 * 2, kind="job",
                 label="CosmoFlow-shaped 16 MiB samples, 128 GiB/rank"),
    "cfg4": dict(D=131072, E=500, N=8, b=64, C=6553, sample_bytes=64 ** 3 * 4, kind="plan",
                 label="AutoPhaseNN-shaped, 5%/rank (40% pooled): 500x500 reuse matrix + ordering"),
    "cfg5": dict(D=1048576, E=1000, N=32, b=512, C=16384, sample_bytes=0, kind="plan", replayers=2,
                 label="1M-id space, logical ranks, 50% pooled buffer"),
}
CFG2 = CONFIGS["cfg2"]
for _c in CONFIGS.values():
    _c.setdefault("seed", 42)
    _c.setdefault("fill_seed", 1)
HBM_BUDGET = 150 * 2 ** 30  # bytes of sample buffers one GPU may hold


def config_for(args) -> dict:
    c = dict(CONFIGS[args.config])
    if args.ranks:  # cfg5 sweep: N logical ranks, C = D / (2N) (50% pooled)
        c["N"] = args.ranks
        if args.config == "cfg5":
            c["C"] = c["D"] // (2 * args.ranks)
    if args.epochs:
        c["E"] = args.epochs
    return c


def workload(name: str, c: dict) -> str:
    sb = c["sample_bytes"]
    size = f", {sb >> 20} MiB samples" if sb >= 1 << 20 else f", {sb >> 10} KiB samples" if sb else ""
    what = "plan+replay+fetch of the whole job" if c["kind"] == "job" else "plan+replay of the whole job"
    return (f"{name}: D={c['D']} E={c['E']} N={c['N']} b={c['b']} C={c['C']} ({c['label']}){size}, {what}")


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_ids: str | None):
        self.idx = gpu_ids  # comma-separated nvidia-smi indices; None = no sampling (ranks > 0)
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                for line in out.splitlines():
                    self.rows.append([c.strip() for c in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        if self.idx is None:
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------- reference --
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


def ref_gather(O, c: dict, warmup: int, steps: int) -> dict:
    """The reference's batch fetch: Store::read_one (store.cpp:134-139) from a
    page-cached store file, on every host core; each step reads one training
    step's global batch (N*b random samples). One store, W + K rounds."""
    SB = c["sample_bytes"]
    B = c["N"] * c["b"]
    count = max(B, min(c["D"], (4 << 30) // SB))  # a store of >= 4 GiB (or the dataset)
    nreads = max(B, (1 << 30) // SB)  # >= 1 GiB per round, so thread start-up is noise
    tmp = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    thr = host_cores()
    out = subprocess.run([O.REF_DUMP, "gather", tmp, str(count), str(SB), str(nreads), str(thr),
                          str(warmup + steps)], check=True, capture_output=True, text=True)
    g = json.loads(out.stdout.strip().splitlines()[-1])
    timed = g["reps"][warmup:]
    g["step_s"] = timed
    g["per_sample_s"] = statistics.median(timed) / nreads
    g["store_samples"] = count
    return g


def ref_planner(O, c: dict, env_extra=None) -> dict:
    """One plan_schedule + simulate_plan pass (pipeline.cpp:32-120,
    buffer.cpp:183-247) of the reference on one host core."""
    cfg = O.Cfg(c["D"], c["E"], c["N"], c["b"], seed=c["seed"], buffer_capacity=c["C"])
    env = dict(os.environ, REF_DUMP_STAGES="0", **(env_extra or {}))
    out = subprocess.run([O.REF_DUMP, "time", "1", *cfg.kv()], check=True, capture_output=True, text=True,
                         env=env).stdout.strip().splitlines()[-1]
    return json.loads(out)


def run_reference(args):
    """The reference's own CPU implementation of the path (oracle/_ref, the
    UNMODIFIED library compiled from /root/reference/proj/src) on this host:
    the planner (single-threaded by construction) on the FULL job once, and the
    Store::read_one batch fetch on every host core, W warm-up + K timed
    steps of one global batch each. value = accesses / (planner seconds +
    accesses x fetch seconds per sample)."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # the checker / reference-arm leg only

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_dump not built "
                          "(needs /root/reference at build time)"}))
        return 0
    c = config_for(args)
    cores = host_cores()
    keep = (c["D"] // (c["N"] * c["b"])) * c["N"] * c["b"]
    A = c["E"] * keep
    # planner: the whole job when it fits the driver's step budget, else
    # (cfg5: hours on one core) E = 1 and 3 and a linear fit in E
    full = args.config != "cfg5"
    if full:
        t = ref_planner(O, c)
        plan_s = t["plan_schedule_s"] + t["simulate_s"]
        psample = f"full job, {t['accesses']} accesses: plan_schedule {t['plan_schedule_s']:.1f} s + " \
                  f"simulate_plan {t['simulate_s']:.1f} s (measured, not extrapolated)"
        same = True
    else:
        pts = []
        for e in (1, 3):
            ce = dict(c, E=e)
            t = ref_planner(O, ce)
            pts.append((e, t["plan_schedule_s"] + t["simulate_s"]))
        slope = (pts[1][1] - pts[0][1]) / 2
        plan_s = pts[0][1] + slope * (c["E"] - 1)
        psample = f"E=1: {pts[0][1]:.1f} s, E=3: {pts[1][1]:.1f} s, linear in E to E={c['E']} " \
                  "(extrapolated: BASELINE.md §3)"
        same = False
    g = ref_gather(O, c, args.warmup, max(args.steps, 1)) if c["sample_bytes"] else None
    gps = g["per_sample_s"] if g else 0.0
    total_s = plan_s + A * gps
    value = A / total_s
    gsample = (f"; fetch: {args.steps} steps of {g['samples']} x Store::read_one of "
               f"{c['sample_bytes']} B from a {g['store_samples']}-sample page-cached store on {g['threads']} "
               f"threads, median {gps * 1e6:.2f} us/sample x {A} accesses") if g else ""
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": workload(args.config, c), "global_batch": c["N"] * c["b"],
                   "parallelism": "reference CPU (planner single-threaded by construction)"},
        "cpu_baseline": {"value": value, "unit": "samples/s",
                         "cores": f"1 (planner) + {cores} (Store::read_one) of {os.cpu_count()} host cores",
                         "kind": "reference", "sample": "planner: " + psample + gsample,
                         "same_config": same},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_stages_s": {"planner_s": plan_s, "fetch_s_per_sample": gps, "fetch_s_job": A * gps},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------------------------ ours --
def host_tier_path(c: dict) -> str:
    d = "/dev/shm" if os.path.isdir("/dev/shm") else "/tmp"
    return os.path.join(d, f"lsg_rows_D{c['D']}_SB{c['sample_bytes']}_s{c['fill_seed']}")


def host_tier_fits(c: dict) -> tuple[bool, str]:
    """The host tier holds the whole dataset's payload rows: it must fit the
    tmpfs and leave most of the host RAM free."""
    need = c["D"] * c["sample_bytes"]
    try:
        avail = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
    except Exception:  # pragma: no cover
        avail = 0
    shm = os.statvfs(os.path.dirname(host_tier_path(c)))
    free = shm.f_bavail * shm.f_frsize
    if need > 0.6 * avail or need > 0.9 * free:
        return False, (f"dataset {need / 2**30:.0f} GiB exceeds the host tier budget "
                       f"({avail / 2**30:.0f} GiB RAM available, {free / 2**30:.0f} GiB tmpfs)")
    return True, ""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--epochs", type=int, default=None, help="override E (debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the one-shot byte check of the fetch")
    ap.add_argument("--plan-shard", default="auto", choices=["auto", "rr", "replicate"],
                    help="N>1: plan each job on one GPU (rr) or on all (replicate); auto = rr above 2 GPUs")
    ap.add_argument("--prio", type=int, default=1, help="plan and replay streams at high priority")
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--ranks", type=int, default=None, help="cfg5: logical ranks (32-256; C = D/(2N))")
    ap.add_argument("--ranks-per-gpu", type=int, default=None,
                    help="diagnostic: fetch only this many of the GPU's ranks (e.g. 1 = the 8-GPU per-GPU shape "
                         "on one GPU); value then counts the fetched ranks' samples")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if os.environ.get("LSG_BENCH_WATCHDOG"):  # debugging: every thread's stack, then exit
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["LSG_BENCH_WATCHDOG"]), exit=True)

    import torch
    import torch.distributed as dist

    import paper_2211_00224_b200 as ls

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    c = config_for(args)
    if c["kind"] == "plan":
        return run_plan_kind(args, c, ls, torch, dist, rank, world, dev)
    D, E, N, b, C, SB = c["D"], c["E"], c["N"], c["b"], c["C"], c["sample_bytes"]
    from paper_2211_00224_b200.parallel import combine_rows, rank_range

    k0, k1 = rank_range(N, world, rank)
    if args.ranks_per_gpu:
        k1 = min(k1, k0 + args.ranks_per_gpu)
    # ranks whose HBM buffers fit on this GPU at once; more ranks per GPU run
    # one group after another through the same buffers (cfg3: 128 GiB/rank)
    per = max(1, min(k1 - k0, HBM_BUDGET // (C * SB)))
    groups = [(g, min(g + per, k1)) for g in range(k0, k1, per)]
    pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, c["seed"], True), buffer_capacity=C)
    sh = pc.shape()
    T, A = int(sh.total_steps), int(sh.total_items)

    # per-rank HBM sample buffers (C slots x sample_bytes) and batch tensors
    bufs = [torch.empty((C, SB), dtype=torch.uint8, device=dev) for _ in range(per)]
    maxlen = min(N * b, max(1024, 2 * b))  # node lists stay near b (checked below)
    outs = [torch.empty((maxlen, SB), dtype=torch.uint8, device=dev) for _ in range(per)]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # the latency-bound stages (the planner's persistent CTA, the per-rank
    # replay CTAs, NCCL) on high-priority streams, the fetch on a low-priority
    # one: the fetch keeps every SM's CTA slots filled (back-to-back step
    # kernels, programmatic dependent launch), so without priority the block
    # scheduler starves the few planner/replay CTAs (measured: plan 0.38 ->
    # 2.0 s beside the fetch); with it they take a slot as soon as one frees
    fstream = torch.cuda.Stream(priority=0)                        # batch fetch
    rstream = torch.cuda.Stream(priority=-1 if args.prio else 0)  # replay + NCCL (lower = higher priority)
    pstream = torch.cuda.Stream(priority=-1 if args.prio else 0)  # plans
    torch.cuda.set_stream(fstream)
    # the loader's pinned staging for the e2e path: two sets, so the plan of
    # job i+1 lands in one while job i's plan is uploaded from the other
    host_sets = [ls.plan_host_buffers(pc) for _ in range(2)] if not args.no_e2e else None

    sh_items = int(sh.total_items)
    # multi-GPU plan placement: "rr" plans job i on GPU i mod N only and
    # broadcasts its node lists; "replicate" plans every job on every GPU
    plan_shard = args.plan_shard == "rr" or (args.plan_shard == "auto" and world > 2)
    # replayed jobs allowed ahead of the fetch: with 4+ GPUs a job's replay
    # (broadcast + replay + row all-gather) is ~0.8x its fetch, and a depth
    # of 2 left a 0.3 s fetch bubble (N=4: 31-33 -> 34.5-34.7 M samples/s)
    ahead = int(os.environ.get("LSG_BENCH_AHEAD", "3" if world > 2 else "2"))
    rr_shift = int(os.environ.get("LSG_BENCH_RR_SHIFT", "0"))  # debug: job i planned on GPU (i + shift) mod N
    # one miss-list / prefetch stream per job in flight: a job's prefetcher
    # holds its stream until the job's misses are consumed
    prep = [torch.cuda.Stream(priority=-1 if args.prio else 0) for _ in range(ahead + 2)]
    ring_bytes = int(float(os.environ.get("LSG_BENCH_RING_GB", "2")) * 2 ** 30)

    # the host tier (e2e miss source): the dataset's Store payload rows in a
    # tmpfs file, pinned; local rank 0 writes it, every process maps it
    hostrows, host_note = None, ""
    if not args.no_e2e and args.steps:
        ok, host_note = host_tier_fits(c)
        if ok:
            path = host_tier_path(c)
            lr = int(os.environ.get("LOCAL_RANK", 0))
            t0 = time.perf_counter()
            if lr == 0:
                hostrows = ls.HostRows(path, D, SB, c["fill_seed"], create=True)
            if world > 1:
                dist.barrier()
            if lr != 0:
                hostrows = ls.HostRows(path, D, SB, c["fill_seed"], create=False)
            host_note = (f"host tier: {D} x {SB} B Store payload rows ({D * SB / 2**30:.0f} GiB) in {path}, "
                         f"pinned + mapped; set up in {time.perf_counter() - t0:.1f} s (outside timing)")

    # the e2e miss ring, shared by consecutive jobs: job i+1's misses (its
    # all-miss first epoch) stream over PCIe into it while job i still fetches
    misses = None
    if hostrows is not None:
        free = torch.cuda.mem_get_info()[0]
        # as much of a job's 64 GiB all-miss first epoch as HBM holds beside the
        # buffers, minus 16 GiB for the jobs in flight (e2e at K=5: 48 GiB
        # 9.17-9.23 M, 59 GiB 9.32-9.47 M, 61 GiB 9.80-9.81 M samples/s; a 12 GiB
        # reserve ran out of memory after 15+ jobs while fetch jobs still took a
        # scratch batch set each)
        want = int(float(os.environ.get("LSG_BENCH_STREAM_GB", "64")) * 2 ** 30)
        reserve = int(float(os.environ.get("LSG_BENCH_RESERVE_GB", "16")) * 2 ** 30)
        ring = max(min(want, free - reserve), 2 * maxlen * per * SB)
        misses = ls.MissStream(SB, ring // SB * SB)
        host_note += f"; miss ring shared across jobs: {ring / 2**30:.1f} GiB"

    def make_jobs(plan, slots, off, host, i):
        """The fetch of job i for every rank group of this GPU (FetchJob:
        miss list, and with the host tier the miss prefetcher, started on a
        prep stream that waits only for this job's replay)."""
        st = prep[i % len(prep)]
        st.wait_stream(torch.cuda.current_stream())
        return [ls.FetchJob(bufs[: g1 - g0], outs[: g1 - g0], (g0, g1), plan, slots, off, SB, c["fill_seed"],
                            host=hostrows if host else None, prep_stream=st, ring_bytes=ring_bytes,
                            misses=misses if host else None)
                for g0, g1 in groups]

    def run_jobs(n, host=False, pipeline=True, stats=None, t_start=None, keep_jobs=False):
        """n passes of the hot path. Job i = plan (K1-K6) -> replay (K7, this
        GPU's ranks, all-gather of the rows) -> fetch (K8 hits from HBM, misses
        from storage, every step of this GPU's ranks), as three pipelined stages on
        three streams:
          planner thread   plans (the step loop is ONE persistent CTA);
          replayer thread  node-list broadcast (N>1, rr placement), replay,
                           the row all-gather (all NCCL calls) and the
                           fetch job's miss list / miss prefetcher;
          this thread      the batch fetch of every step.
        With `pipeline` job i+1's plan and replay overlap job i's fetch on the
        remaining SMs; every job's work is complete when the call returns.
        With the rr placement job i is planned once, on GPU i mod N, and its
        node lists are broadcast over NVLink: jobs are independent units, so
        the plan stream shards across GPUs although one plan's step
        recurrence does not. host=True is the e2e path: the plan lands in
        pinned host memory (lsg_plan_host) and is uploaded by its GPU, the
        hit/miss rows are read back to the host, and misses are read from the
        host tier over PCIe."""
        import queue
        qp, qr = queue.Queue(maxsize=1), queue.Queue(maxsize=1)
        free = threading.Semaphore(2)
        fetched = threading.Semaphore(ahead if pipeline else 1)  # replayed jobs ahead of the fetch
        err = []
        shard = world > 1 and plan_shard
        mine = [i for i in range(n) if not shard or (i + rr_shift) % world == rank]
        tj0 = time.perf_counter()
        plan_evs = []

        def planner():
            try:
                torch.cuda.set_device(dev)  # the CUDA current device is per host thread
                with torch.cuda.stream(pstream):
                    if t_start is not None:
                        pstream.wait_event(t_start)
                    for j, i in enumerate(mine):
                        free.acquire()
                        a, z = ev(), ev()
                        a.record(pstream)
                        out = (ls.plan_schedule_host(pc, buffers=host_sets[j % 2]) if host
                               else ls.plan_schedule(pc))
                        z.record(pstream)
                        plan_evs.append((i, a, z))
                        qp.put((out, a, z))
                        if not pipeline:
                            z.synchronize()
            except BaseException as e:  # surfaced on the main thread
                err.append(e)
                qp.put(None)

        rows = []

        def replayer():
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(rstream):
                    if t_start is not None:
                        rstream.wait_event(t_start)
                    for i in range(n):
                        owner = (i + rr_shift) % world if shard else rank
                        pa = pz = None
                        if owner == rank:
                            got = qp.get()
                            if got is None:
                                raise err[0]
                            out, pa, pz = got
                            rstream.wait_event(pz)
                            plan = out.plan
                            if host:  # the plan lives in host memory: upload for the replay
                                items = plan.items.to(dev, non_blocking=True)
                                noff = plan.node_off.to(dev, non_blocking=True)
                            else:  # device outputs of the plan stream
                                items, noff = plan.items, plan.node_off
                                for t in (items, noff):
                                    t.record_stream(rstream)
                        else:
                            items = torch.empty(sh_items, dtype=torch.int32, device=dev)
                            noff = torch.empty((T, N + 1), dtype=torch.int32, device=dev)
                        fetched.acquire()
                        f0 = ev()
                        f0.record(rstream)
                        if shard:  # the owner's node lists to every GPU
                            dist.broadcast(items, src=owner)
                            dist.broadcast(noff, src=owner)
                        fb = ev()
                        fb.record(rstream)
                        plan = ls.SchedulePlan(D, N, b, int(sh.steps_per_epoch), None, items, noff, None, None)
                        h0 = time.perf_counter()
                        sim = ls.simulate_plan(plan, C, node_range=(k0, k1), want_slots=True)
                        h1 = time.perf_counter()
                        combine_rows(sim.hits, sim.misses)
                        if host:  # d2h of the step results
                            rows.append((ls.to_host(sim.hits), ls.to_host(sim.misses)))
                        off = ls.to_host(noff).numpy()
                        if int((off[:, k0 + 1:k1 + 1] - off[:, k0:k1]).max()) > maxlen:
                            raise SystemExit("a node list exceeds the batch tensor rows")
                        if os.environ.get("LSG_BENCH_TIMELINE"):
                            print(f"[replayer] rank {rank} n={n} job {i} t0={1e3 * (h0 - tj0):.1f}: simulate_plan {1e3 * (h1 - h0):.1f} ms host, "
                                  f"rows+off {1e3 * (time.perf_counter() - h1):.1f} ms", file=sys.stderr, flush=True)
                        if owner == rank:
                            free.release()  # this job's host staging set has been uploaded
                        f1 = ev()
                        f1.record(rstream)
                        jobs = make_jobs(plan, sim.slots, off, host, i)
                        if os.environ.get("LSG_BENCH_TIMELINE") and t_start is not None:
                            f1.synchronize()
                            print(f"[replay-gpu] rank {rank} job {i}: start {t_start.elapsed_time(f0):.1f} "
                                  f"bcast-done {t_start.elapsed_time(fb):.1f} end {t_start.elapsed_time(f1):.1f}",
                                  file=sys.stderr, flush=True)
                        for t in (items, noff, sim.slots):
                            t.record_stream(fstream)
                        qr.put((plan, sim, off, pa, pz, f0, f1, jobs))
            except BaseException as e:
                err.append(e)
                qr.put(None)

        ths = [threading.Thread(target=planner, daemon=True), threading.Thread(target=replayer, daemon=True)]
        for th in ths:
            th.start()
        for i in range(n):
            got = qr.get()
            if got is None:
                raise err[0]
            plan, sim, off, pa, pz, f0, f1, jobs = got
            fstream.wait_event(f1)
            f1b = ev()
            f1b.record(fstream)
            for job in jobs:  # rank groups one after another (shared buffers)
                job.run()
            f2 = ev()
            f2.record(fstream)
            if stats is not None:
                stats.append((pa, pz, f0, f1, f2, sim, off, f1b, jobs if keep_jobs else None, plan))
            if not keep_jobs:
                for job in jobs:  # stream-ordered free after the job's kernels (rings, lists)
                    job.close(fstream)
            if not pipeline:
                f2.synchronize()
            fetched.release()
        for th in ths:
            th.join()
        if os.environ.get("LSG_BENCH_TIMELINE") and t_start is not None:
            for i, a, z in plan_evs:
                z.synchronize()
                print(f"[plan-gpu] rank {rank} job {i}: {t_start.elapsed_time(a):.1f} -> {t_start.elapsed_time(z):.1f}",
                      file=sys.stderr, flush=True)
        return rows

    # warm-up (also the first pass that fills the HBM buffers)
    nwarm = max(args.warmup, 3 if args.steps else 0)
    if nwarm and world > 1 and plan_shard:
        # every GPU plans at least one warm-up job: a GPU's FIRST plan
        # allocates its output tensors (cudaMalloc), which waited for the
        # NCCL broadcast kernel spinning on that GPU, doubling the plan of
        # job world-1 inside the timed region (4 GPUs: 380 -> 680-800 ms)
        nwarm = max(nwarm, world)
    if nwarm:
        run_jobs(nwarm)
    torch.cuda.synchronize()

    # hit/miss totals of the local ranks (for algorithmic bytes), from the
    # fetch jobs' own counts
    st0 = []
    run_jobs(1, stats=st0, keep_jobs=True)
    torch.cuda.synchronize()
    fst = [j.stats() for j in st0[0][8]]
    for j in st0[0][8]:
        j.close(fstream)
    local_hits = sum(s["hits"] for s in fst)
    local_misses = sum(s["misses"] for s in fst)
    kept_local = sum(s["kept"] for s in fst)
    assert local_hits == int(st0[0][5].hits[:, k0:k1].sum()) and local_misses == int(st0[0][5].misses[:, k0:k1].sum())
    keep_plan = st0[0]  # plan, replay and offsets of one job, for the byte check below
    del st0

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ls.lib().lsg_launch_count()
    # rank 0 samples every GPU of the job with ONE nvidia-smi process (the
    # line it prints carries the clocks of all of them)
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    nloc = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    gpu_ids = ",".join(vis.split(",")[:nloc] if vis else [str(g) for g in range(nloc)])
    evs = []
    with ClockSampler(gpu_ids if rank == 0 else None) as clk:
        t_start, t_end = ev(), ev()
        t_start.record(fstream)
        run_jobs(args.steps, stats=evs, t_start=t_start)
        t_end.record(fstream)
        torch.cuda.synchronize()
    launches = ls.lib().lsg_launch_count() - launches0
    total_ms = t_start.elapsed_time(t_end)
    # per-job stage windows on rank 0 (ms from t_start), read after the timed region
    timeline = [[round(t_start.elapsed_time(x), 1) if x is not None else None for x in (e[0], e[1], e[2], e[3], e[7], e[4])]
                for e in evs]
    own = [e[0].elapsed_time(e[1]) for e in evs if e[0] is not None]
    plan_ms = statistics.mean(own) if own else 0.0
    replay_ms = statistics.mean(e[2].elapsed_time(e[3]) for e in evs)
    fetch_ms = statistics.mean(e[7].elapsed_time(e[4]) for e in evs)
    del evs
    # one job alone (no overlap): the latency of a single plan+replay+fetch pass
    serial, sst = [], []
    if args.steps:
        a0, a1 = ev(), ev()
        if world > 1:
            dist.barrier()
        a0.record(fstream)
        run_jobs(1, pipeline=False, t_start=a0, stats=sst)
        a1.record(fstream)
        torch.cuda.synchronize()
        serial.append(a0.elapsed_time(a1))
    job_ms = serial[0] if serial else 0.0
    # the plan of that job alone (nothing beside it): the plan's own latency
    plan_alone_ms = sst[0][0].elapsed_time(sst[0][1]) if sst and sst[0][0] is not None else 0.0
    del sst
    if world > 1:
        tt = torch.tensor([total_ms, plan_ms, replay_ms, fetch_ms, job_ms, plan_alone_ms], device=dev,
                          dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, plan_ms, replay_ms, fetch_ms, job_ms, plan_alone_ms = [float(x) for x in tt]
    ms_per_step = total_ms / max(args.steps, 1)
    # samples of one job: the whole job, or (diagnostic --ranks-per-gpu) the
    # fetched ranks' rows on every GPU
    A_job = A if not args.ranks_per_gpu else (local_hits + local_misses) * world

    # HBM-gather algorithmic bytes: hits read a slot and write the batch row
    # (SURVEY §8d); misses come from storage and are reported apart
    hit_bytes = 2 * SB * local_hits
    miss_bytes = SB * local_misses + SB * kept_local  # batch row + kept slot writes
    achieved = hit_bytes / (fetch_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = traffic_ratio = None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "gather_traffic.json")))
        traffic = tr.get("dram_bytes_per_launch")
        traffic_ratio = tr.get("dram_bytes_per_byte_algorithmic")
    except Exception:
        pass

    # e2e through the public API with host buffers: the plan lands in pinned
    # host memory (lsg_plan_host) and is uploaded for the replay, hit/miss rows
    # are read back, and every miss is read from the host tier over PCIe (the
    # TMA miss prefetcher); the same pipelined job stream, K jobs
    e2e = None
    if not args.no_e2e and args.steps:
        run_jobs(2, host=True)  # untimed warm-up of the host path
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = ev(), ev()
        est = []
        a0.record(fstream)
        run_jobs(args.steps, host=True, t_start=a0, stats=est)
        a1.record(fstream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(a1) / args.steps
        e2e_fetch_ms = statistics.mean(e[7].elapsed_time(e[4]) for e in est)
        e2e_timeline = [[round(a0.elapsed_time(x), 1) for x in (e[7], e[4])] for e in est]
        host_bytes = local_misses * SB if hostrows is not None else 0  # every miss read once from the host tier
        del est
        if world > 1:
            tt = torch.tensor([e2e_ms, e2e_fetch_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms, e2e_fetch_ms = float(tt[0]), float(tt[1])
            hb = torch.tensor([host_bytes], device=dev, dtype=torch.int64)
            dist.all_reduce(hb)
            host_bytes = int(hb[0])
        d2h = A * 4 * 2 + T * (N + 1) * 4 + 2 * T * N * 4 * 2 + E * E * 8 + E * 4 + 8 + 4 \
            + pc.pso.max_iters * 8 + T * N * 4 * 2 + T * (N + 1) * 4
        e2e = {"value": A / (e2e_ms * 1e-3), "unit": "samples/s",
               "h2d_bytes_per_step": T * (N + 1) * 4 + A * 4 + host_bytes,
               "d2h_bytes_per_step": d2h,
               "miss_source": ("host tier over PCIe (TMA prefetcher)" if hostrows is not None else
                               "Store payload synthesised on device: " + host_note),
               "pcie": ({"miss_bytes_per_job": host_bytes,
                         "achieved_gbs": host_bytes / (e2e_fetch_ms * 1e-3) / 1e9 / max(world, 1),
                         "fetch_ms": e2e_fetch_ms,
                         "note": "per GPU: host-tier bytes / fetch-phase time (the PCIe reads overlap the HBM "
                                 "gather; epoch 0 is all misses)"} if hostrows is not None else None),
               "fetch_windows_ms": e2e_timeline,
               "note": "per job: lsg_plan_host (trace, graph, order, plan lists, fetch counts to pinned host), "
                       "plan re-uploaded for the replay, hit/miss rows read back, batch fetch with every miss "
                       "read from storage; jobs pipelined as in value" + ("; " + host_note if host_note else "")}

    # one-shot byte check of the benched fetch (off the timed region): the
    # job's batches at evenly spaced steps equal Store::read_one of their ids
    verify = None
    if not args.no_verify and args.steps:
        verify = verify_fetch(ls, torch, keep_plan, groups, bufs, outs, SB, c["fill_seed"], hostrows, T)
    del keep_plan
    cpu = cpu_baseline(c, args.config) if (rank == 0 and world == 1) else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": A_job / (ms_per_step * 1e-3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (splitmix64 traces and Store payload, seed 42 / fill_seed 1)",
            "config": {"workload": workload(args.config, c),
                       "global_batch": N * b, "ranks_per_gpu": k1 - k0, "rank_groups": len(groups),
                       "parallelism": (f"jobs' plans round-robin over {world} GPUs (node lists broadcast, NCCL); "
                                       if world > 1 and plan_shard else
                                       "plan replicated per GPU; " if world > 1 else "")
                                      + f"replay+fetch sharded {k1 - k0} ranks/GPU",
                       "l2": f"inputs > L2 ({C * SB / 2**30:.1f} GiB HBM sample buffer per rank)"},
            "pipeline": "plan / replay / fetch on three streams: later jobs' plans (1 persistent CTA) and replays "
                        "overlap job i's fetch; every job's full work is inside the timed region; "
                        "value: misses written from the Store payload synthesised on device",
            "plan_ms": plan_ms, "replay_ms": replay_ms, "fetch_ms": fetch_ms,
            "single_job_ms": job_ms, "single_job_samples_per_s": A / (job_ms * 1e-3) if job_ms else None,
            "plan_alone_ms": plan_alone_ms,
            "plan_samples_per_s": A / (plan_alone_ms * 1e-3) if plan_alone_ms else A / (plan_ms * 1e-3),
            "plan_samples_per_s_note": "one plan (shuffle+order+evict+assign of the whole job) alone; plan_ms is "
                                       "the mean plan time inside the pipeline, beside other jobs' fetch",
            "gather": {"value": achieved, "unit": "GB/s", "hits": local_hits, "misses": local_misses,
                       "kept_misses": kept_local, "hit_bytes_per_job": hit_bytes,
                       "miss_bytes_per_job": miss_bytes,
                       "all_bytes_gbs": (hit_bytes + miss_bytes) / (fetch_ms * 1e-3) / 1e9,
                       "note": "HBM gather = 2 x sample_bytes per hit over the fetch phase (the misses' time "
                               "included, their bytes not: SURVEY §8d)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_note": "dram read+write bytes per k_fetch_fused launch (one steady-state step, "
                                         "8 ranks on one GPU) from profiles/gather_traffic.json (r02f_fetch_final.ncu-rep); "
                                         f"{traffic_ratio:.3f} x that launch's algorithmic bytes" if traffic else None,
                         "kernel": "fetch phase (k_fetch_fused: persistent multi-step TMA bulk-copy pipeline, "
                                   "producer/consumer warps: hits, misses and deferred slot fills)",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if peaks else "fallback 6650"},
            "gpu_launches": int(launches),
            **({"timeline_plan0_plan1_rep0_rep1_fetch0_fetch1": timeline} if timeline else {}),
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if verify:
            line["verify"] = verify
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
    if misses is not None:
        misses.close()
    if hostrows is not None:
        hostrows.close()
        if world > 1:
            dist.barrier()
        if int(os.environ.get("LOCAL_RANK", 0)) == 0:
            try:
                os.remove(host_tier_path(c))
            except OSError:
                pass
    if world > 1:
        dist.destroy_process_group()
    return 0


def verify_fetch(ls, torch, kept, groups, bufs, outs, SB, fill_seed, hostrows, T, npts=24):
    """Byte check of the fetch at the bench shape: one planned+replayed job
    fetched in segments (the same FetchJob path as the timed region), and
    after each segment every batch row of its last step compared with the
    Store payload of its id (store.cpp:134-139, via K9 store_fill). Runs the
    device-synthesised miss path and, with a host tier, the PCIe miss path."""
    sim, off, plan = kept[5], kept[6], kept[9]
    pts = sorted({max(0, int(T * (i + 1) / npts) - 1) for i in range(npts)})
    items = plan.items
    N = off.shape[1] - 1
    bases = np.concatenate([[0], np.cumsum(off[:, N].astype(np.int64))])
    out = {"steps_checked": 0, "rows_checked": 0, "mismatched_rows": 0, "paths": []}
    for path, host in (("misses synthesised on device", None), ("misses from the host tier", hostrows)):
        if path.endswith("tier") and host is None:
            continue
        out["paths"].append(path)
        for g0, g1 in groups:
            prev = 0
            for g in pts:
                j = ls.FetchJob(bufs[: g1 - g0], outs[: g1 - g0], (g0, g1), plan, sim.slots, off, SB, fill_seed,
                                host=host, step_range=(prev, g + 1))
                j.run()
                j.close()
                prev = g + 1
                ids = items[bases[g]: bases[g + 1]] & 0x7FFFFFFF
                for k in range(g0, g1):
                    lo, hi = int(off[g, k]), int(off[g, k + 1])
                    if hi == lo:
                        continue
                    want = ls.store_fill(ids[lo:hi], SB, fill_seed)
                    bad = int((outs[k - g0][: hi - lo] != want).any(dim=1).sum())
                    out["rows_checked"] += hi - lo
                    out["mismatched_rows"] += bad
                out["steps_checked"] += 1
    torch.cuda.synchronize()
    if out["mismatched_rows"]:
        raise SystemExit(f"fetch byte check FAILED: {out}")
    return out


def run_plan_kind(args, c, ls, torch, dist, rank, world, dev):
    """cfg4 / cfg5: the plan (K1-K6) + replay (K7) of the whole job, K jobs
    per GPU (independent jobs, weak scaling; job j+1's plan overlaps job j's
    replay). value = planned-and-replayed samples of all GPUs / timed region
    (max over ranks)."""
    D, E, N, b, C = c["D"], c["E"], c["N"], c["b"], c["C"]
    pc = ls.PipelineConfig(trace=ls.TraceConfig(D, E, N, b, c["seed"], True), buffer_capacity=C)
    sh = pc.shape()
    A = int(sh.total_items)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    st = torch.cuda.current_stream()

    def one():
        a, m, z = ev(), ev(), ev()
        a.record(st)
        out = ls.plan_schedule(pc)
        m.record(st)
        sim = ls.simulate_plan(out.plan, C)
        z.record(st)
        return a, m, z, out, sim

    for _ in range(args.warmup):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = ls.lib().lsg_launch_count()
    res = []
    # jobs are independent: job j+1's plan (a planner thread on its own
    # stream; the plan loop holds one small cluster) overlaps the replays of
    # earlier jobs (one CTA per rank), two replayer threads on their own streams
    import queue
    import threading
    # (cfg5's replay outlasts its plan: two replays in flight, 62 -> 91 M samples/s at K=5; cfg4 is
    # plan-bound and a second replay only slows its plan)
    nrep = max(1, int(os.environ.get("LSG_BENCH_REPLAYERS", str(c.get("replayers", 1)))))
    ps = torch.cuda.Stream(device=dev)
    rss = [torch.cuda.Stream(device=dev) for _ in range(nrep)]
    with ClockSampler(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] if rank == 0 else None) as clk:
        t0, t1 = ev(), ev()
        t0.record(st)
        q, err = queue.Queue(maxsize=1), []

        def planner():
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(ps):
                    ps.wait_event(t0)
                    for _ in range(args.steps):
                        a, m = ev(), ev()
                        a.record(ps)
                        out = ls.plan_schedule(pc)
                        m.record(ps)
                        q.put((out, a, m))
            except BaseException as e:  # surfaced on the main thread
                err.append(e)
                for _ in range(nrep):
                    q.put(None)

        lock = threading.Lock()
        left = [args.steps]

        def replayer(rs):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(rs):
                    rs.wait_event(t0)
                    while True:
                        with lock:
                            if left[0] == 0:
                                return
                            left[0] -= 1
                        got = q.get()
                        if got is None:
                            return
                        out, a, m = got
                        rs.wait_event(m)
                        for t in (out.plan.items, out.plan.node_off):
                            t.record_stream(rs)
                        z = ev()
                        sim = ls.simulate_plan(out.plan, C)
                        z.record(rs)
                        with lock:
                            res.append((a, m, z))
                        del out, sim
            except BaseException as e:  # surfaced on the main thread
                err.append(e)

        th = threading.Thread(target=planner)
        th.start()
        reps = [threading.Thread(target=replayer, args=(rs,)) for rs in rss]
        for r in reps:
            r.start()
        th.join()
        for r in reps:
            r.join()
        if err:
            raise err[0]
        for rs in rss:
            st.wait_stream(rs)
        t1.record(st)
        torch.cuda.synchronize()
    launches = ls.lib().lsg_launch_count() - launches0
    total_ms = t0.elapsed_time(t1)
    plan_ms = statistics.mean(a.elapsed_time(m) for a, m, z in res)
    replay_ms = statistics.mean(m.elapsed_time(z) for a, m, z in res)
    # the HBM-bound stage that is callable alone: K1 (trace + inverse
    # permutations): 4 B per emitted index
    tr = []
    for _ in range(3):
        a, z = ev(), ev()
        a.record(st)
        ls.generate_trace(pc.trace)
        z.record(st)
        torch.cuda.synchronize()
        tr.append(a.elapsed_time(z))
    k1_ms = min(tr)
    if world > 1:
        tt = torch.tensor([total_ms, plan_ms, replay_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, plan_ms, replay_ms = [float(x) for x in tt]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    k1_gbs = 4 * A / (k1_ms * 1e-3) / 1e9
    cpu = cpu_baseline(c, args.config) if (rank == 0 and world == 1) else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": world * args.steps * A / (total_ms * 1e-3), "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (splitmix64 traces, seed 42)",
            "config": {"workload": workload(args.config, c), "global_batch": N * b,
                       "parallelism": f"independent jobs, {args.steps} per GPU" if world > 1 else "one GPU",
                       "l2": "trace and next-use arrays > L2"},
            "plan_ms": plan_ms, "replay_ms": replay_ms,
            "pipeline": f"job j+1's plan (planner thread, own stream) beside the replays of earlier jobs "
                        f"({nrep} replayer threads, own streams)",
            "plan_samples_per_s": A / (plan_ms * 1e-3),
            "roofline": {"bound": "hbm", "achieved": k1_gbs, "peak": peak, "unit": "GB/s", "frac": k1_gbs / peak,
                         "traffic": None, "kernel": "K1 shuffle (generate_trace: 4 B per emitted index; the plan "
                                                    "and replay are latency-bound step recurrences)"},
            "gpu_launches": int(launches), "clocks": clk.summary(),
            "e2e": None,
        }
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_baseline(c: dict, name: str):
    """The reference CPU planner (oracle/_ref) on a bounded sample of the
    job (~10-20 s of one core: the first E_s epochs) plus Store::read_one on
    all host cores; rank 0 at N=1 only. The bench's reference arm times the
    full job."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import oracle as O
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    if not O.ref_available():
        return {"value": None, "unit": "samples/s", "cores": 1, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}
    es = min(c["E"], 10 if name in ("cfg2", "cfg4") else 3 if name == "cfg5" else c["E"])
    ce = dict(c, E=es)
    t = ref_planner(O, ce)
    g = ref_gather(O, c, 1, 3) if c["sample_bytes"] else None
    per = (t["plan_schedule_s"] + t["simulate_s"]) / t["accesses"] + (g["per_sample_s"] if g else 0.0)
    return {"value": 1.0 / per, "unit": "samples/s",
            "cores": f"1 (planner) + {host_cores()} (Store::read_one) of {os.cpu_count()} host cores",
            "kind": "reference",
            "sample": f"{name} shape, first E={es} of {c['E']} epochs ({t['accesses']} accesses): plan_schedule "
                      f"{t['plan_schedule_s']:.2f} s + simulate_plan {t['simulate_s']:.2f} s"
                      + (f"; Store::read_one of {c['sample_bytes']} B: {g['per_sample_s'] * 1e6:.2f} us/sample "
                         f"on {g['threads']} threads (median of 3 global batches)" if g else ""),
            "plan_samples_per_s": t["accesses"] / t["plan_schedule_s"]}


if __name__ == "__main__":
    sys.exit(main())
