#!/usr/bin/env python
"""bench.py — candidate plans evaluated/sec of the B200 plan-evaluation engine.

Workload (BASELINE.json configs[4], the largest; fits one GPU because no plan
list is materialised): constrained_search over the C5 1024-GPU cluster
(24x16 H800 + 24x16 H20 + 16x16 PCIe-class, 70B policy, L=80) for the 1023-device
three-type train set -> 2,415,919,104 candidate layouts per step, window 3.
One step = one full pass over that candidate space (stage-table build + layout
scan + argmin). At N GPUs the rank space is split into N contiguous shards
(strong scaling), and the per-shard (cost, rank) winners are all-gathered over
NCCL and reduced lexicographically (the only collective).

value : candidates/s with the train set resident on the device (device time of
        the stage tables + scan, CUDA events on the engine's stream, max over ranks)
e2e   : the same metric through the public C ABI with host buffers:
        gp_constrained_search_range (host prep + H2D + kernels + D2H) + the NCCL
        all-gather, timed on the device.
Inputs are tiny (~0.5 MB of tables), so L2 is flushed (a 512 MiB write)
between timed steps.

--impl reference: the reference's own constrained_search (oracle/_ref, compiled
from /root/reference by oracle/Makefile) on the host cores, one thread per core
(cap 32), on bounded C5 train sets (its plan list is materialised in RAM).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CONFIG = "c5_1024gpu"
WINDOW = 3
METRIC = "candidate plans evaluated/sec"
# from the committed ncu capture of K1-fast on this workload (profiles/r01/)
K1_PROFILE = "profiles/r02/k1_layout_scan_fast_ncu_summary.txt"
K1_WARP_INST_PER_CAND = 4.160   # smsp__inst_executed.sum / candidates (10,050,744,126 / 2,415,919,104)
K1_DRAM_BYTES_PER_LAUNCH = 1629440  # dram__bytes_read.sum + dram__bytes_write.sum (tables + middle rows, L2-resident)
UNIT = "plans/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), \
        int(os.environ.get("WORLD_SIZE", 1))


def problem():
    from common import problem as load
    return load(CONFIG)


def bench_train_set(p):
    return list(range(p.cluster.n - 1))


def cpu_sample_sets(p, count):
    """Bounded C5 train sets for the reference (which materialises every layout):
    16 H800 machines + 8 H20 machines -> 36,864 layouts, 384 devices each,
    rotated over the cluster's machines."""
    cl = p.cluster
    by_type = {}
    for m, t in enumerate(cl.machine_type.tolist()):
        by_type.setdefault(t, []).append(m)
    sets = []
    for i in range(count):
        h800 = by_type[0][i % 8: i % 8 + 16]
        h20 = by_type[1][(3 * i) % 16: (3 * i) % 16 + 8]
        ms = set(h800 + h20)
        sets.append([d for d in range(cl.n) if cl.device_machine[d] in ms])
    return sets


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index: int):
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- reference
def ref_threads():
    """Host threads the --impl reference arm uses (one bounded set per thread per step)."""
    return max(1, min(os.cpu_count() or 1, 32))


def ref_rate(p, sets, threads, window=WINDOW, with_costs=False):
    import ctypes as C

    import numpy as np
    from oracles import Ref, ref_available
    if not ref_available():
        return None
    ref = Ref(p)
    lib = ref.lib
    lib.ref_bench_constrained_search.argtypes = [C.c_void_p, C.POINTER(C.c_int32),
                                                 C.POINTER(C.c_int32), C.c_int, C.c_int, C.c_int,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double)]
    flat = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.int32) for s in sets]))
    lens = np.asarray([len(s) for s in sets], dtype=np.int32)
    secs, chk = C.c_double(), C.c_double()
    costs = np.zeros(len(sets), dtype=np.float64)
    rc = lib.ref_bench_constrained_search(ref.h, flat.ctypes.data_as(C.POINTER(C.c_int32)),
                                          lens.ctypes.data_as(C.POINTER(C.c_int32)), len(sets),
                                          window, threads, C.byref(secs), C.byref(chk),
                                          costs.ctypes.data_as(C.POINTER(C.c_double)))
    if rc:
        raise RuntimeError(lib.ref_last_error().decode())
    if with_costs:
        return secs.value, costs.tolist()
    return secs.value


def cpu_baseline(p, threads=1, n_sets=12):
    """Reference (oracle/_ref) on the host cores, bounded sample; port (oracle/) if absent."""
    from oracles import Oracle, ref_available
    sets = cpu_sample_sets(p, n_sets)
    orc = Oracle(p)
    layouts = sum(orc.train_space(s) for s in sets)
    sample = f"{n_sets} C5 train sets x 36,864 layouts (16 H800 + 8 H20 machines, 384 devices), window {WINDOW}"
    if ref_available():
        secs = ref_rate(p, sets, threads)
        kind = "reference"
    else:
        t = time.perf_counter()
        for s in sets:
            orc.constrained_search(s, WINDOW)
        secs = time.perf_counter() - t
        kind = "port"
        threads = 1
    return {"value": layouts / secs, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": sample, "seconds": secs, "cpu": cpu_model(), "nproc": os.cpu_count()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    p = problem()
    threads = ref_threads()
    sets = cpu_sample_sets(p, threads)
    from oracles import Oracle, ref_available
    orc = Oracle(p)
    layouts = sum(orc.train_space(s) for s in sets)
    kind = "reference" if ref_available() else "port"
    times = []
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            secs = ref_rate(p, sets, threads)
        else:
            t = time.perf_counter()
            for s in sets:
                orc.constrained_search(s, WINDOW)
            secs = time.perf_counter() - t
        if i >= args.warmup:
            times.append(secs)
    total = sum(times)
    value = layouts * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{CONFIG}: reference constrained_search, bounded sample of "
                               f"{len(sets)} train sets x 36,864 layouts (one per host thread)",
                   "window": WINDOW},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads if kind == "reference" else 1,
                         "kind": kind, "sample": f"{len(sets)} C5 train sets x 36,864 layouts per step",
                         "cpu": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- B200
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2511_00796_b200.engine import Engine

    rank, local_rank, world = dist_env()
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    p = problem()
    ids = bench_train_set(p)
    eng = Engine(p, device=local_rank)
    total = eng.train_space(ids)
    from paper_2511_00796_b200.shard import gather_winner
    # balanced contiguous rank shards, cut where every shard keeps K1-fast's scan order
    bounds = eng.shard_bounds(ids, world)
    lo, hi = bounds[rank], bounds[rank + 1]
    stream = torch.cuda.ExternalStream(eng.stream_ptr, device=dev)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def gather(res):
        """All-gather (cost, rank, feasible) of every shard; lexicographic min (shard.py)."""
        return gather_winner(bool(res.found), res.cost, res.rank, res.feasible, device=dev)

    # ---- device-resident timing (value) ------------------------------------
    eng.set_timing(True)
    eng.train_prepare(ids)
    for _ in range(args.warmup):
        eng.train_launch(WINDOW, lo, hi)
        eng.train_collect()
    sampler = ClockSampler(local_rank) if rank == 0 else None
    dev_ms, k1_ms, k2_ms = [], [], []
    res = None
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.train_launch(WINDOW, lo, hi)
        b.record(stream)
        res, _ = eng.train_collect()
        dev_ms.append(a.elapsed_time(b))
        k2, k1 = eng.train_timing()
        k2_ms.append(k2)
        k1_ms.append(k1)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop() if sampler else None
    win = gather(res)
    # ---- end-to-end through the public C ABI with host buffers (e2e) --------
    h2d0, d2h0, _ = eng.io_bytes()
    e2e_ms = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        r2, _ = eng.constrained_search_raw(ids, WINDOW, lo=lo, hi=hi)
        g = gather(r2)
        b.record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e_ms.append(a.elapsed_time(b))
    h2d1, d2h1, sum_stages = eng.io_bytes()
    steps_e2e = args.warmup + args.steps
    h2d_step = (h2d1 - h2d0) / steps_e2e
    d2h_step = (d2h1 - d2h0) / steps_e2e + 24 * world

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t_dev = max_over_ranks(sum(dev_ms))
    t_e2e = max_over_ranks(sum(e2e_ms))
    t_k1 = max_over_ranks(sum(k1_ms))
    t_k2 = max_over_ranks(sum(k2_ms))
    launches = eng.launches
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    best = win if win[1] >= 0 else None
    value = total * args.steps / (t_dev / 1e3)
    e2e = total * args.steps / (t_e2e / 1e3)
    # ---- roofline of the dominant kernel (K1 layout scan) -------------------
    # K1-fast is an integer / table-gather kernel: per candidate
    # a 32-byte suffix record, rank-count and promotion-table lookups in shared memory, two
    # (max total, max compute) reads, ~6 fp64 adds/muls. No tensor-core or HBM bound
    # applies (its tables stay in L2/L1: ~1 MB DRAM per launch), so it is reported against
    # the SM instruction-issue roofline: warp instructions per candidate (ncu, constant for
    # this code and workload) x candidates/s vs 4 issue slots/clk/SM x SMs x SM clock.
    k1_s = t_k1 / 1e3 / args.steps
    shard = hi - lo
    props = torch.cuda.get_device_properties(dev)
    sm_mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    peak_issue = 4 * props.multi_processor_count * sm_mhz * 1e6
    achieved = K1_WARP_INST_PER_CAND * shard / k1_s
    avg_S = sum_stages / total
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_dev / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{CONFIG}: constrained_search over the 1023-device 3-type train set "
                               f"(24x16 H800 + 24x16 H20 + 15x16+15 PCIe), 70B L=80, window {WINDOW}",
                   "candidates_per_step": total, "parallelism": f"rank-range shards x{world}",
                   "l2": "flushed (512 MiB write) between timed steps"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d_step),
                "d2h_bytes_per_step": int(d2h_step), "ms_per_step": t_e2e / args.steps},
        "roofline": {"bound": "issue", "achieved": achieved / 1e12, "peak": peak_issue / 1e12,
                     "unit": "Twarp-inst/s", "frac": achieved / peak_issue,
                     "traffic": K1_DRAM_BYTES_PER_LAUNCH * shard / total,
                     "kernel": "k1_layout_scan_fast", "warp_inst_per_candidate": K1_WARP_INST_PER_CAND,
                     "counts_from": K1_PROFILE, "avg_stages": avg_S,
                     "k1_ms_per_step": t_k1 / args.steps, "k2_ms_per_step": t_k2 / args.steps,
                     "peak_source": f"4 issue slots/clk/SM x {props.multi_processor_count} SMs x "
                                    f"{sm_mhz:.0f} MHz (median SM clock sampled in the timed region)"},
        "gpu_launches": launches,
        "clocks": clocks,
        "winner": {"cost": best[0], "rank": int(best[1])} if best else None,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(p)
    if not args.no_units:
        line["units"] = {"U1_same_workload": same_workload(local_rank, args.steps, args.warmup),
                         "U2_milp": milp_rate(local_rank), "U3_partition": partition_rate(local_rank)}
    if not args.no_ttp:  # (at N > 1: rank 0 alone, one multi-GPU context over all N devices)
        line["time_to_best_plan"] = time_to_best_plan(list(range(world)) if world > 1 else [local_rank])
    print(json.dumps(line), flush=True)
    return 0


def same_workload(device, steps, warmup):
    """U1 like-for-like with the reference arm: the SAME bounded C5 train sets the
    --impl reference arm scans on this host (one per host thread), through the public batched
    entry point gp_constrained_search_batch (host buffers: one H2D, all sets in flight, one
    D2H; memo off so every step scans), and the per-set costs checked against the
    reference's own constrained_search on those sets."""
    import torch

    from paper_2511_00796_b200.engine import Engine
    from oracles import Oracle, ref_available
    p = problem()
    sets = cpu_sample_sets(p, ref_threads())
    layouts = sum(Oracle(p).train_space(s) for s in sets)
    out = {"sets": len(sets), "layouts_per_step": layouts, "window": WINDOW,
           "sample": f"{len(sets)} C5 train sets x 36,864 layouts (the --impl reference workload)"}
    with Engine(p, device=device) as eng:
        eng.set_memo(False)
        secs = []
        for i in range(warmup + steps):
            torch.cuda.synchronize(device)
            t = time.perf_counter()
            res = eng.constrained_search_batch_raw(sets, WINDOW)
            torch.cuda.synchronize(device)
            if i >= warmup:
                secs.append(time.perf_counter() - t)
        launches = eng.launches
    gpu_costs = [r.cost if r.found else -1.0 for r, _ in res]
    out["b200_e2e"] = {"value": layouts / statistics.median(secs), "unit": UNIT,
                       "ms_per_step": 1e3 * statistics.median(secs), "kernel_launches": launches}
    if ref_available():
        rsecs, rcosts = ref_rate(p, sets, ref_threads(), with_costs=True)
        out["reference_cpu"] = {"value": layouts / rsecs, "unit": UNIT, "threads": ref_threads(),
                                "seconds": rsecs}
        out["speedup_e2e"] = out["b200_e2e"]["value"] / out["reference_cpu"]["value"]
        out["costs_identical"] = gpu_costs == rcosts
    return out


def milp_rate(device):
    """U2: MILP state x config relaxations/s of solve_milp (src/rollout_milp.cpp:115-142) on
    a C5 rollout set with a 5e6-state capacity lattice (a fresh context: no cached lattice),
    beside the reference's own solve_milp on a 1e6-state lattice on one host core. Work =
    sum over configs c of the lattice states where c fits (one DADD + DSETP each)."""
    import torch

    from paper_2511_00796_b200.engine import Engine
    from oracles import Ref, ref_available
    p = problem()
    cl = p.cluster

    def rollout(per_type):
        out = []
        for t in range(len(cl.type_names)):
            out += [d for d in range(cl.n) if cl.device_type[d] == t][:per_type]
        return sorted(out)

    def relax(cfgs, caps):
        tot = 0
        for c in cfgs:
            v = [c["type_counts"][t] if isinstance(c, dict) else c.type_counts[t] for t in range(len(caps))]
            prod = 1
            for t, cap in enumerate(caps):
                prod *= max(0, cap - v[t] + 1)
            tot += prod
        return tot

    out = {}
    roll = rollout(170)
    B = float(p.workload.batch_rollouts * WINDOW)
    secs = []
    for _ in range(3):
        with Engine(p, device=device) as eng:
            cfgs = eng.enumerate_configs(roll)
            caps = eng.rollout_capacities(roll)
            eng.solve_milp(eng.enumerate_configs(rollout(20)), eng.rollout_capacities(rollout(20)), B,
                           p.workload.mean_len)  # warm the context (another lattice)
            torch.cuda.synchronize(device)
            t = time.perf_counter()
            res, _ = eng.solve_milp(cfgs, caps, B, p.workload.mean_len)
            torch.cuda.synchronize(device)
            secs.append(time.perf_counter() - t)
    states = 1
    for c in caps:
        states *= c + 1
    work = relax(cfgs, caps)
    out["b200"] = {"value": work / min(secs), "unit": "relaxations/s", "lattice_states": states,
                   "configs": len(cfgs), "relaxations": work, "seconds": min(secs),
                   "makespan": res.makespan}
    if ref_available():
        ref = Ref(p)
        small = rollout(100)
        cfg = ref.enumerate_configs(small)
        t = time.perf_counter()
        ref.solve_milp(cfg["configs"], cfg["capacities"], B, p.workload.mean_len)
        rs = time.perf_counter() - t
        rstates = 1
        for c in cfg["capacities"]:
            rstates *= c + 1
        rw = relax(cfg["configs"], cfg["capacities"])
        out["reference_cpu"] = {"value": rw / rs, "unit": "relaxations/s", "lattice_states": rstates,
                                "configs": len(cfg["configs"]), "seconds": rs, "threads": 1}
        out["speedup"] = out["b200"]["value"] / out["reference_cpu"]["value"]
    return out


def partition_rate(device):
    """U3: move/swap candidates examined per second by graph_partition_candidates
    (src/partition.cpp:284-349, 16 restarts, top-8) at N = 1024 (band [0.45, 0.55]); the
    work count comes from the C restatement's identical local search (or_partition_evals),
    the result is checked against the reference's own call, timed on one host core."""
    import torch

    from paper_2511_00796_b200 import abi
    from paper_2511_00796_b200.engine import Engine
    from oracles import Oracle, Ref, oracle_partitions, ref_available
    p = problem()
    lo, hi, seed = 0.45, 0.55, 4276115
    orc = Oracle(p)
    orc.lib.or_partition_evals.restype = __import__("ctypes").c_int64
    orc.lib.or_partition_evals(1)
    want = oracle_partitions(orc, lo, hi, seed=seed)
    evals = orc.lib.or_partition_evals(1)
    o = abi.gp_part_opts(12, 16, seed, 1e-9, 0, 0)
    with Engine(p, device=device) as eng:
        eng.partition_candidates(0.2, 0.3, k=8, opts=o)  # unit tables, first launches
        secs = []
        for _ in range(3):
            torch.cuda.synchronize(device)
            t = time.perf_counter()
            got = eng.partition_candidates(lo, hi, k=8, opts=o)
            torch.cuda.synchronize(device)
            secs.append(time.perf_counter() - t)
    out = {"band": [lo, hi], "restarts": 16, "k": 8, "move_swap_evals": evals,
           "b200": {"value": evals / min(secs), "unit": "move/swap gains/s", "seconds_per_call": min(secs)},
           "matches_restatement": got == want}
    if ref_available():
        t = time.perf_counter()
        r = Ref(p).partition_candidates(lo, hi, k=8, seed=seed)
        rs = time.perf_counter() - t
        out["reference_cpu"] = {"value": evals / rs, "unit": "move/swap gains/s", "seconds_per_call": rs,
                                "threads": 1}
        out["speedup"] = rs / min(secs)
        out["matches_reference"] = got == [(c["train"], c["objective"], c["compute_fraction"])
                                           for c in r["candidates"]]
    return out


def time_to_best_plan(devices, keys=("c3_64gpu/eta=1", "c4_256gpu/eta=2", "c5_1024gpu/eta=2")):
    """schedule() wall time (all window passes, up to the final plan) through the native
    batched driver (gp_schedule) on a freshly created context over `devices` (one GPU, or
    a multi-GPU context at N > 1: train batches split by layout count, MILP batches by
    configuration list); context setup excluded, like the reference's input loading. The
    reference's own schedule() on one host core for the configs it can finish (plans compared
    field by field); the C4 plan is compared with the C restatement's whole-schedule fixture."""
    from common import problem as load
    from oracles import Ref, ref_available

    from paper_2511_00796_b200.engine import Engine
    out = {}
    for key in keys:
        name, eta = key.split("/eta=")
        prob = load(name)
        kw = {"devices": list(devices)} if len(devices) > 1 else {"device": devices[0]}
        with Engine(prob, **kw) as eng:  # warm-up run: CUDA module load, first allocations
            eng.schedule(eta=int(eta), seed=4276115)
        with Engine(prob, **kw) as eng:
            t = time.perf_counter()
            plan, _ = eng.schedule(eta=int(eta), seed=4276115)
            b200_s = time.perf_counter() - t
        row = {"b200_s": b200_s, "gpus": len(devices), "window": plan["window_steps"],
               "objective": max(plan["costs"]["train_s"], plan["costs"]["infer_total_s"])}
        if name in ("c1_desk_mixed", "c2_16gpu", "c3_64gpu") and ref_available():
            t = time.perf_counter()
            ref = json.loads(Ref(prob).schedule(eta=int(eta))["plan_json"])
            row["reference_cpu_s"] = time.perf_counter() - t
            for k in ("format", "cluster_fingerprint", "calibration_fingerprint", "workload_fingerprint"):
                ref.pop(k, None)
            row["plan_identical"] = ref == plan
        elif name == "c4_256gpu":
            # the reference's own C4 schedule() takes 6.6 h on one core: run once offline
            # (tests/golden/make_golden_c4_reference.py), its plan and wall time committed
            from common import golden
            r = golden("schedule_c4_reference.json")["c4_256gpu/eta=2"]
            row["reference_cpu_s"] = r["reference_seconds"]
            row["reference_cpu_s_source"] = "tests/golden/schedule_c4_reference.json (one core, build container)"
            row["plan_identical"] = plan == r["plan"]
            g = golden("schedule_c4_oracle.json")["c4_256gpu/eta=2"]
            row["c_restatement_cpu_s"] = g["oracle_seconds"]
        elif name == "c5_1024gpu":
            row["reference_cpu_s"] = "infeasible: materialises 4.3e11 layouts per pass (SURVEY.md 8a A5)"
        out[key] = row
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttp", action="store_true", help="skip the time-to-best-plan runs")
    ap.add_argument("--no-units", action="store_true",
                    help="skip the same-workload / MILP / partition unit measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
