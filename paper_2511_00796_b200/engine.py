"""Python host binding of libgplan.so — mirrors the reference's free-function API
(inc/train_search.hpp:29, inc/rollout_milp.hpp:22-37, inc/cost_model.hpp:63,
inc/partition.hpp:40-55) with the same argument meaning and error behaviour:
ValidationError / InfeasibleError / BandInfeasibleError are raised where the
reference throws them, and `constrained_search` returns None for std::nullopt.

There is no CPU fallback: constructing an Engine without the built library or
without an sm_100 GPU raises EngineUnavailable.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import abi
from .inputs import Problem

_LIB_PATH = os.environ.get("GPLAN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                       "libgplan.so")
_lib = None


class EngineUnavailable(RuntimeError):
    pass


class ValidationError(ValueError):
    pass


class InfeasibleError(RuntimeError):
    pass


class BandInfeasibleError(InfeasibleError):
    pass


class CapacityError(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise EngineUnavailable(
                f"{_LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        _lib = C.CDLL(_LIB_PATH)
        abi.declare(_lib, "gp")
        _lib.gp_ctx_destroy.argtypes = [C.c_void_p]
        _lib.gp_ctx_launches.argtypes = [C.c_void_p]
        _lib.gp_ctx_launches.restype = C.c_longlong
        vp = C.c_void_p
        _lib.gp_ctx_stream.argtypes = [vp]
        _lib.gp_ctx_stream.restype = vp
        _lib.gp_train_prepare.argtypes = [vp, abi.i32p, C.c_int32, C.POINTER(abi.gp_train_opts)]
        _lib.gp_train_launch.argtypes = [vp, C.c_int32, C.c_int64, C.c_int64]
        _lib.gp_train_collect.argtypes = [vp, C.POINTER(abi.gp_train_result), abi.i32p]
        _lib.gp_ctx_set_timing.argtypes = [vp, C.c_int]
        _lib.gp_ctx_set_memo.argtypes = [vp, C.c_int]
        _lib.gp_solve_milp_batch.argtypes = [vp, C.c_int32, C.POINTER(abi.gp_config), abi.i32p, abi.i32p,
                                             C.c_int32, abi.f64p, C.c_double, C.POINTER(abi.gp_rollout_result),
                                             C.POINTER(abi.gp_rollout_entry), abi.i32p]
        _lib.gp_train_timing.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]
        _lib.gp_ctx_io_bytes.argtypes = [vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
                                         C.POINTER(C.c_double)]
        _lib.gp_ctx_io_bytes.restype = None
        _lib.gp_fp64_peak.argtypes = [vp, C.POINTER(C.c_double)]
    return _lib


def _check(rc: int) -> None:
    if rc == abi.GP_OK:
        return
    msg = lib().gp_last_error().decode()
    if rc == abi.GP_INVALID:
        raise ValidationError(msg)
    if rc == abi.GP_BAND_INFEASIBLE:
        raise BandInfeasibleError(msg)
    if rc == abi.GP_INFEASIBLE:
        raise InfeasibleError(msg)
    if rc == abi.GP_CAPACITY:
        raise CapacityError(msg)
    raise EngineUnavailable(f"CUDA error: {msg}")


def _ids(ids) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(ids, dtype=np.int32))


@dataclass
class Stage:
    devices: list
    tp: int
    dp: int
    layers: int


@dataclass
class TrainSearchResult:
    stages: list
    cost: float
    rank: int
    layouts: int
    feasible: int


class Engine:
    """One engine context (cluster + workload + calibration uploaded to one GPU)."""

    def __init__(self, problem: Problem, device: int = 0, devices=None):
        """devices: list of CUDA ordinals for an in-call multi-GPU context (searches fan out)."""
        self.problem = problem
        self.n_devices = problem.cluster.n
        c, w, k = problem.structs()
        self._structs = (c, w, k)
        h = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*devices)
            lib().gp_ctx_create_multi.argtypes = [C.POINTER(abi.gp_cluster), C.POINTER(abi.gp_workload),
                                                  C.POINTER(abi.gp_calib), C.POINTER(C.c_int), C.c_int,
                                                  C.POINTER(C.c_void_p)]
            _check(lib().gp_ctx_create_multi(C.byref(c), C.byref(w), C.byref(k), arr, len(devices),
                                             C.byref(h)))
        else:
            _check(lib().gp_ctx_create(C.byref(c), C.byref(w), C.byref(k), device, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().gp_ctx_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def launches(self) -> int:
        return int(lib().gp_ctx_launches(self._h))

    # ---- training side ------------------------------------------------------
    def train_space(self, train_set, opts: abi.gp_train_opts | None = None) -> int:
        ids = _ids(train_set)
        out = C.c_int64()
        _check(lib().gp_train_space(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                    C.byref(opts or abi.default_train_opts()), C.byref(out)))
        return out.value

    def constrained_search_raw(self, train_set, window: int, opts=None, lo: int = 0, hi: int = -1):
        ids = _ids(train_set)
        res = abi.gp_train_result()
        devs = np.zeros(max(len(ids), 1), dtype=np.int32)
        o = opts or abi.default_train_opts()
        if lo == 0 and hi < 0:
            rc = lib().gp_constrained_search(self._h, ids.ctypes.data_as(abi.i32p), len(ids), window,
                                             C.byref(o), C.byref(res), devs.ctypes.data_as(abi.i32p))
        else:
            rc = lib().gp_constrained_search_range(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                                   window, C.byref(o), lo, hi, C.byref(res),
                                                   devs.ctypes.data_as(abi.i32p))
        _check(rc)
        return res, devs

    def constrained_search_batch_raw(self, train_sets, window: int, opts=None):
        """Many constrained_search calls in one (gp_constrained_search_batch): returns
        [(gp_train_result, stage devices array)] in input order."""
        off = np.zeros(len(train_sets) + 1, dtype=np.int32)
        for i, t in enumerate(train_sets):
            off[i + 1] = off[i] + len(t)
        ids = np.ascontiguousarray(np.concatenate([np.asarray(t, dtype=np.int32) for t in train_sets])
                                   if train_sets else np.zeros(1, dtype=np.int32))
        res = (abi.gp_train_result * max(len(train_sets), 1))()
        devs = np.zeros(max(int(off[-1]), 1), dtype=np.int32)
        _check(lib().gp_constrained_search_batch(self._h, len(train_sets), ids.ctypes.data_as(abi.i32p),
                                                 off.ctypes.data_as(abi.i32p), window,
                                                 C.byref(opts or abi.default_train_opts()), res,
                                                 devs.ctypes.data_as(abi.i32p)))
        return [(res[i], devs[off[i]:off[i + 1]]) for i in range(len(train_sets))]

    def constrained_search(self, train_set, window: int, opts=None, lo: int = 0, hi: int = -1):
        """constrained_search (inc/train_search.hpp:29-33); None == std::nullopt."""
        res, devs = self.constrained_search_raw(train_set, window, opts, lo, hi)
        if not res.found:
            return None
        stages = []
        for s in range(res.n_stages):
            st = res.stage[s]
            stages.append(Stage(devs[st.first:st.first + st.count].tolist(), st.tp, st.dp, st.layers))
        return TrainSearchResult(stages, res.cost, res.rank, res.layouts, res.feasible)

    def debug_layout_costs(self, train_set, lo: int, hi: int, path: int = 0, opts=None):
        """Test hook: per_step of every layout of ranks [lo, hi) as the scan kernel computes it
        (+inf: memory-infeasible). path 0 = the whole-space scan a search runs, 1 = generic K1,
        2 = K1-fast with every candidate deferred, 3 = K1-fast over the range as a range search.
        Returns (array, fast_used) with fast_used = 1 + K1-fast's inner run, 0 = generic."""
        ids = _ids(train_set)
        out = np.empty(max(hi - lo, 1), dtype=np.float64)
        fast = C.c_int32()
        _check(lib().gp_debug_layout_costs(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                           C.byref(opts or abi.default_train_opts()), lo, hi, path,
                                           out.ctypes.data_as(abi.f64p), C.byref(fast)))
        return out[:hi - lo], fast.value

    def shard_bounds(self, train_set, n_shards: int, opts=None):
        """Rank boundaries of n_shards balanced contiguous shards (gp_train_shard_bounds)."""
        ids = _ids(train_set)
        b = np.zeros(n_shards + 1, dtype=np.int64)
        _check(lib().gp_train_shard_bounds(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                           C.byref(opts or abi.default_train_opts()), n_shards,
                                           b.ctypes.data_as(C.POINTER(C.c_int64))))
        return b.tolist()

    # ---- split form + measurement hooks (bench.py) -------------------------
    @property
    def stream_ptr(self) -> int:
        return int(lib().gp_ctx_stream(self._h))

    def train_prepare(self, train_set, opts=None):
        self._prep_ids = _ids(train_set)
        _check(lib().gp_train_prepare(self._h, self._prep_ids.ctypes.data_as(abi.i32p),
                                      len(self._prep_ids), C.byref(opts or abi.default_train_opts())))

    def train_launch(self, window: int, lo: int = 0, hi: int = -1):
        _check(lib().gp_train_launch(self._h, window, lo, hi))

    def train_collect(self):
        res = abi.gp_train_result()
        devs = np.zeros(max(len(self._prep_ids), 1), dtype=np.int32)
        _check(lib().gp_train_collect(self._h, C.byref(res), devs.ctypes.data_as(abi.i32p)))
        return res, devs

    def train_candidates_search(self, train_set, window: int):
        """Product-space training search (enumerate_train_candidates x train_plan_fits x
        train_step_cost, first minimum; tests/oracles.cpp:166-174) -> (gp_train_result, devices).
        res.layouts = candidates, res.rank = the winner's candidate index."""
        ids = _ids(train_set)
        res = abi.gp_train_result()
        devs = np.zeros(max(len(ids), 1), dtype=np.int32)
        _check(lib().gp_train_candidates_search(self._h, ids.ctypes.data_as(abi.i32p), len(ids), window,
                                                C.byref(res), devs.ctypes.data_as(abi.i32p)))
        return res, devs

    def exhaustive(self, window: int):
        """exhaustive_schedule_optimum (tests/oracles.cpp:144-209) over every bipartition."""
        out = abi.gp_exhaustive_result()
        ids = np.zeros(self.problem.cluster.n, dtype=np.int32)
        _check(lib().gp_exhaustive_optimum(self._h, window, C.byref(out), ids.ctypes.data_as(abi.i32p)))
        return {"feasible": bool(out.feasible), "objective": out.objective if out.feasible else None,
                "train_set": ids[:out.n_train].tolist(), "partitions": out.partitions,
                "train_candidates": out.train_candidates, "replica_vectors": out.replica_vectors}

    def solve_milp_batch(self, queries, B, mean_len=None):
        """queries: [(configs (list of gp_config), caps)] -> [(status, gp_rollout_result, entries)]."""
        mean_len = self.problem.workload.mean_len if mean_len is None else mean_len
        dims = len(self.problem.cluster.type_names)
        off = [0]
        for cfgs, _ in queries:
            off.append(off[-1] + len(cfgs))
        allc = (abi.gp_config * max(off[-1], 1))(*[c for cfgs, _ in queries for c in cfgs])
        offs = np.array(off, dtype=np.int32)
        caps = np.array([list(c) for _, c in queries], dtype=np.int32).reshape(-1)
        Bs = np.full(len(queries), float(B))
        out = (abi.gp_rollout_result * max(len(queries), 1))()
        ent = (abi.gp_rollout_entry * max(off[-1], 1))()
        st = np.zeros(max(len(queries), 1), dtype=np.int32)
        _check(lib().gp_solve_milp_batch(self._h, len(queries), allc, offs.ctypes.data_as(abi.i32p),
                                         caps.ctypes.data_as(abi.i32p), dims,
                                         Bs.ctypes.data_as(abi.f64p), mean_len, out, ent,
                                         st.ctypes.data_as(abi.i32p)))
        res = []
        for i in range(len(queries)):
            n = out[i].n_entries if st[i] == 0 else 0
            res.append((int(st[i]), out[i], [ent[off[i] + k] for k in range(n)]))
        return res

    def simulate(self, plan: dict, steps: int, seeds, sync_every: int = 1):
        """simulate (src/simulator.cpp:381-403) of a plan document (plan_to_json form) under
        this context's workload with the plan's staleness, one GPU thread per seed.
        Returns ([report dict per seed], used rollout devices)."""
        cl, w = self.problem.cluster, self.problem.workload
        T = len(cl.type_names)
        ents = plan["rollout_plan"]["entries"]
        cfgs = (abi.gp_config * max(len(ents), 1))()
        reps = np.zeros(max(len(ents), 1), dtype=np.int32)
        for i, e in enumerate(ents):
            for t in range(T):
                cfgs[i].type_counts[t] = e["type_counts"][t]
            cfgs[i].n_stages = len(e["tp_per_stage"])
            for s, tp in enumerate(e["tp_per_stage"]):
                cfgs[i].tp[s] = tp
            cfgs[i].throughput = e["throughput_tps"]
            reps[i] = e["replicas"]
        train = _ids(plan["partition"]["train"])
        roll = _ids(plan["partition"]["rollout"])
        price = np.ascontiguousarray(cl.type_price[np.asarray(cl.device_type)], dtype=np.float64)
        blen = np.array([int(l) for l, _ in w.histogram], dtype=np.int32)
        bprob = np.array([float(p) for _, p in w.histogram], dtype=np.float64)
        c = plan["costs"]
        sp = abi.gp_sim_plan(int(plan["window_steps"]), int(plan["staleness"]), c["train_s"], c["update_s"],
                             c["reward_s"], len(ents), cfgs, reps.ctypes.data_as(abi.i32p), len(train),
                             len(roll), train.ctypes.data_as(abi.i32p), roll.ctypes.data_as(abi.i32p),
                             price.ctypes.data_as(abi.f64p), len(blen), blen.ctypes.data_as(abi.i32p),
                             bprob.ctypes.data_as(abi.f64p))
        seeds = np.asarray(list(seeds), dtype=np.uint64)
        out = (abi.gp_sim_report * max(len(seeds), 1))()
        used = np.zeros(max(len(roll), 1), dtype=np.int32)
        n_used = C.c_int32()
        _check(lib().gp_simulate(self._h, C.byref(sp), steps, sync_every,
                                 seeds.ctypes.data_as(C.POINTER(C.c_uint64)), len(seeds), out,
                                 used.ctypes.data_as(abi.i32p), C.byref(n_used)))
        reports = []
        for i in range(len(seeds)):
            r = {f: getattr(out[i], f) for f, _ in abi.gp_sim_report._fields_ if f != "pad"}
            if r["dollar_cost_per_token"] != r["dollar_cost_per_token"]:
                r["dollar_cost_per_token"] = None
            reports.append(r)
        return reports, used[:n_used.value].tolist()

    def set_memo(self, on: bool = True):
        """Enable (default) / disable + drop the window-independent constrained_search memo."""
        _check(lib().gp_ctx_set_memo(self._h, int(on)))

    def set_timing(self, on: bool = True):
        _check(lib().gp_ctx_set_timing(self._h, int(on)))

    def train_timing(self):
        k2, k1 = C.c_float(), C.c_float()
        _check(lib().gp_train_timing(self._h, C.byref(k2), C.byref(k1)))
        return k2.value, k1.value

    def io_bytes(self):
        h2d, d2h, ss = C.c_longlong(), C.c_longlong(), C.c_double()
        lib().gp_ctx_io_bytes(self._h, C.byref(h2d), C.byref(d2h), C.byref(ss))
        return h2d.value, d2h.value, ss.value

    def fp64_peak(self) -> float:
        v = C.c_double()
        _check(lib().gp_fp64_peak(self._h, C.byref(v)))
        return v.value

    # ---- rollout side ---------------------------------------------------------
    def enumerate_configs(self, rollout_set, opts=None, cap: int = 4096):
        """enumerate_configs (inc/rollout_milp.hpp:22-25) -> list of gp_config."""
        ids = _ids(rollout_set)
        out = (abi.gp_config * cap)()
        n = C.c_int32()
        _check(lib().gp_enumerate_configs(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                          C.byref(opts or abi.default_rollout_opts()), out, cap,
                                          C.byref(n)))
        return [out[i] for i in range(n.value)]

    def rollout_capacities(self, rollout_set):
        ids = _ids(rollout_set)
        caps = np.zeros(len(self.problem.cluster.type_names), dtype=np.int32)
        _check(lib().gp_rollout_capacities(self._h, ids.ctypes.data_as(abi.i32p), len(ids),
                                           caps.ctypes.data_as(abi.i32p)))
        return caps.tolist()

    def solve_milp(self, configs, caps, total_rollouts: float, mean_len: float):
        """solve_milp (inc/rollout_milp.hpp:35-37) -> (gp_rollout_result, [gp_rollout_entry])."""
        arr = (abi.gp_config * max(len(configs), 1))(*configs)
        caps = _ids(caps)
        res = abi.gp_rollout_result()
        ent = (abi.gp_rollout_entry * max(len(configs), 1))()
        _check(lib().gp_solve_milp(self._h, arr, len(configs), caps.ctypes.data_as(abi.i32p),
                                   len(caps), total_rollouts, mean_len, C.byref(res), ent))
        return res, [ent[i] for i in range(res.n_entries)]

    def weight_sync_cost(self, train, rollout, entry_types, entry_replicas, window: int) -> float:
        t, r = _ids(train), _ids(rollout)
        et, er = _ids(entry_types), _ids(entry_replicas)
        out = C.c_double()
        _check(lib().gp_weight_sync_cost(self._h, t.ctypes.data_as(abi.i32p), len(t),
                                         r.ctypes.data_as(abi.i32p), len(r),
                                         et.ctypes.data_as(abi.i32p), er.ctypes.data_as(abi.i32p),
                                         len(et), window, C.byref(out)))
        return out.value

    # ---- repartition ----------------------------------------------------------
    def partition_candidates(self, gamma_l: float, gamma_h: float, k: int = 8, opts=None,
                             q: float = 0.0, r: float = 1.0):
        """graph_partition_candidates (inc/partition.hpp:53-55): [(train ids, objective, fraction)]."""
        g = abi.gp_gamma(q, r, gamma_l, gamma_h)
        out = (abi.gp_partition * k)()
        ids = np.zeros(self.n_devices * k, dtype=np.int32)
        n = C.c_int32()
        _check(lib().gp_partition_candidates(self._h, C.byref(g), C.byref(opts or abi.default_part_opts()),
                                             k, out, ids.ctypes.data_as(abi.i32p), C.byref(n)))
        return [(ids[o.train_offset:o.train_offset + o.train_count].tolist(), o.objective,
                 o.compute_fraction) for o in out[:n.value]]

    def partition_objective(self, train):
        t = _ids(train)
        obj, frac = C.c_double(), C.c_double()
        _check(lib().gp_partition_objective(self._h, t.ctypes.data_as(abi.i32p), len(t), C.byref(obj),
                                            C.byref(frac)))
        return obj.value, frac.value

    # ---- Algorithm-1 driver -----------------------------------------------------
    def schedule(self, eta: int = -1, seed: int = 0x5EED, expand_window: bool = True, restarts: int = 16,
                 with_stats: bool = False):
        """schedule() (inc/scheduler.hpp:53-54) on the engine. Returns the plan_to_json fields
        (src/plan_io.cpp:43-75, values only, no fingerprints) plus the iteration trace."""
        L = lib()
        L.gp_default_sched_opts.argtypes = [C.POINTER(abi.gp_sched_opts)]
        L.gp_default_sched_opts.restype = None
        o = abi.gp_sched_opts()
        L.gp_default_sched_opts(C.byref(o))
        o.eta_override, o.seed, o.expand_window, o.restarts = eta, seed, int(expand_window), restarts
        N = self.n_devices
        res = abi.gp_schedule_result()
        tr = np.zeros(N, dtype=np.int32)
        ro = np.zeros(N, dtype=np.int32)
        sd = np.zeros(N, dtype=np.int32)
        cap = 8 * 70
        cfg = (abi.gp_config * cap)()
        ent = (abi.gp_rollout_entry * cap)()
        trace = np.zeros(4 * o.iteration_cap, dtype=np.float64)
        L.gp_schedule.argtypes = [C.c_void_p, C.POINTER(abi.gp_sched_opts), C.POINTER(abi.gp_schedule_result),
                                  abi.i32p, abi.i32p, abi.i32p, C.POINTER(abi.gp_config),
                                  C.POINTER(abi.gp_rollout_entry), C.c_int32, abi.f64p]
        _check(L.gp_schedule(self._h, C.byref(o), C.byref(res), tr.ctypes.data_as(abi.i32p),
                             ro.ctypes.data_as(abi.i32p), sd.ctypes.data_as(abi.i32p), cfg, ent, cap,
                             trace.ctypes.data_as(abi.f64p)))
        T = len(self.problem.cluster.type_names)
        t = res.train
        plan = {
            "window_steps": res.window, "staleness": res.staleness, "iterations_run": res.iterations_run,
            "converged": bool(res.converged),
            "partition": {"train": tr[:res.n_train].tolist(), "rollout": ro[:res.n_rollout].tolist()},
            "train_plan": {"stages": [{"devices": sd[s.first:s.first + s.count].tolist(), "tp": s.tp,
                                       "dp": s.dp, "layers": s.layers} for s in t.stage[:t.n_stages]],
                           "cost_s": t.cost},
            "rollout_plan": {"entries": [{"type_counts": list(cfg[i].type_counts[:T]),
                                          "tp_per_stage": list(cfg[i].tp[:cfg[i].n_stages]),
                                          "throughput_tps": cfg[i].throughput,
                                          "machine_footprint": list(cfg[i].tp[:cfg[i].n_stages]),
                                          "replicas": ent[i].replicas, "workload_rollouts": ent[i].workload}
                                         for i in range(res.rollout.n_entries)],
                             "makespan_s": res.rollout.makespan, "total_rollouts": res.rollout.total_rollouts},
            "costs": {"train_s": res.c_train, "rollout_s": res.c_rollout, "reward_s": res.c_reward,
                      "update_s": res.c_update, "infer_total_s": res.c_infer_total, "window_steps": res.window},
        }
        tr_rows = trace[:4 * res.n_trace].reshape(-1, 4).tolist()
        if with_stats:
            return plan, tr_rows, {"evaluated_partitions": res.evaluated_partitions,
                                   "evaluated_layouts": res.evaluated_layouts}
        return plan, tr_rows
