"""Test-side access to the checkers (TEST INFRASTRUCTURE ONLY).

* liboracle.so — the plain-C restatement in oracle/ (always buildable, travels).
* libref.so    — the UNMODIFIED reference compiled from /root/reference by
                 oracle/Makefile (present only where it was built).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from paper_2511_00796_b200 import abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_ref", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref.so")

_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        _oracle = C.CDLL(ORACLE_SO)
        abi.declare(_oracle, "or")
        _oracle.or_schedule.argtypes = [C.POINTER(abi.gp_cluster), C.POINTER(abi.gp_workload),
                                        C.POINTER(abi.gp_calib), C.c_void_p, C.POINTER(C.c_void_p)]
        _oracle.or_free.argtypes = [C.c_void_p]
        P = C.POINTER
        _oracle.or_layout_costs.argtypes = [P(abi.gp_cluster), P(abi.gp_workload), P(abi.gp_calib),
                                            abi.i32p, C.c_int32, P(abi.gp_train_opts), C.c_int64,
                                            C.c_int64, P(C.c_double)]
        _oracle.or_layout_costs_tab.argtypes = [P(abi.gp_cluster), P(abi.gp_workload), P(abi.gp_calib),
                                                abi.i32p, C.c_int32, P(abi.gp_train_opts), C.c_int32,
                                                P(C.c_int64), P(C.c_int64), P(C.c_double)]
        _oracle.or_constrained_search_tab.argtypes = [
            P(abi.gp_cluster), P(abi.gp_workload), P(abi.gp_calib), abi.i32p, C.c_int32,
            P(abi.gp_train_opts), abi.i32p, C.c_int32, C.c_int64, C.c_int64, C.c_int32,
            P(C.c_double), P(C.c_int64), P(C.c_int64), P(C.c_int64), P(C.c_double)]
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_SO)
        vp, cp = C.c_void_p, C.c_char_p
        P = C.POINTER
        _ref.ref_ctx_create.argtypes = [cp, cp, cp, P(vp)]
        _ref.ref_ctx_destroy.argtypes = [vp]
        _ref.ref_last_error.restype = cp
        _ref.ref_free.argtypes = [vp]
        _ref.ref_ctx_describe.argtypes = [vp, P(vp)]
        _ref.ref_schedule.argtypes = [vp, C.c_int, C.c_ulonglong, C.c_int, C.c_int, P(vp)]
        _ref.ref_constrained_search.argtypes = [vp, abi.i32p, C.c_int, C.c_int, C.c_int, C.c_int, P(vp)]
        _ref.ref_train_candidates.argtypes = [vp, abi.i32p, C.c_int, C.c_int, P(vp)]
        _ref.ref_enumerate_configs.argtypes = [vp, abi.i32p, C.c_int, C.c_int, P(vp)]
        _ref.ref_solve_milp.argtypes = [cp, abi.i32p, C.c_int, C.c_double, C.c_double, P(vp)]
        _ref.ref_weight_sync.argtypes = [vp, abi.i32p, C.c_int, abi.i32p, C.c_int, C.c_int, cp,
                                         P(C.c_double)]
        _ref.ref_exhaustive_optimum.argtypes = [vp, C.c_int, P(vp)]
        _ref.ref_simulate.argtypes = [vp, cp, C.c_int, C.c_ulonglong, C.c_int, P(vp)]
        _ref.ref_brute_milp.argtypes = [cp, abi.i32p, C.c_int, C.c_double, C.c_double, P(vp)]
        _ref.ref_partition_candidates.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_double,
                                                  C.c_int, C.c_ulonglong, C.c_int, C.c_int, C.c_int,
                                                  P(vp)]
        _ref.ref_partition_objective.argtypes = [vp, abi.i32p, C.c_int, P(C.c_double), P(C.c_double)]
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ids(ids):
    return np.ascontiguousarray(np.asarray(ids, dtype=np.int32))


class Ref:
    """The unmodified reference library on one (cluster, workload, calibration)."""

    def __init__(self, problem):
        self.lib = ref_lib()
        c, w, k = problem.texts
        h = C.c_void_p()
        rc = self.lib.ref_ctx_create(c.encode(), w.encode(), (k or "").encode(), C.byref(h))
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_ctx_destroy(self.h)

    def _json(self, rc, out):
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())
        s = C.cast(out, C.c_char_p).value.decode()
        self.lib.ref_free(out)
        return json.loads(s)

    def describe(self):
        out = C.c_void_p()
        return self._json(self.lib.ref_ctx_describe(self.h, C.byref(out)), out)

    def schedule(self, eta=-1, seed=4276115, expand=True, restarts=16):
        out = C.c_void_p()
        return self._json(self.lib.ref_schedule(self.h, eta, seed, int(expand), restarts,
                                                C.byref(out)), out)

    def constrained_search(self, ids, window, max_per_type=4, gran=16):
        ids = _ids(ids)
        out = C.c_void_p()
        return self._json(self.lib.ref_constrained_search(
            self.h, ids.ctypes.data_as(abi.i32p), len(ids), window, max_per_type, gran,
            C.byref(out)), out)

    def train_candidates(self, ids, window):
        ids = _ids(ids)
        out = C.c_void_p()
        return self._json(self.lib.ref_train_candidates(self.h, ids.ctypes.data_as(abi.i32p),
                                                        len(ids), window, C.byref(out)), out)

    def exhaustive(self, window):
        out = C.c_void_p()
        return self._json(self.lib.ref_exhaustive_optimum(self.h, window, C.byref(out)), out)

    def simulate(self, plan_json, steps, seed, sync_every=1):
        out = C.c_void_p()
        rc = self.lib.ref_simulate(self.h, plan_json.encode(), steps, seed, sync_every, C.byref(out))
        return self._json(rc, out)

    def brute_milp(self, configs, caps, B, mean_len):
        caps = _ids(caps)
        out = C.c_void_p()
        rc = self.lib.ref_brute_milp(json.dumps(configs).encode(), caps.ctypes.data_as(abi.i32p),
                                     len(caps), B, mean_len, C.byref(out))
        return self._json(rc, out)

    def enumerate_configs(self, ids, max_stages=4):
        ids = _ids(ids)
        out = C.c_void_p()
        return self._json(self.lib.ref_enumerate_configs(self.h, ids.ctypes.data_as(abi.i32p),
                                                         len(ids), max_stages, C.byref(out)), out)

    def solve_milp(self, configs, caps, B, mean_len):
        caps = _ids(caps)
        out = C.c_void_p()
        rc = self.lib.ref_solve_milp(json.dumps(configs).encode(), caps.ctypes.data_as(abi.i32p),
                                     len(caps), B, mean_len, C.byref(out))
        return self._json(rc, out)

    def weight_sync(self, train, roll, window, rollout_plan):
        t, r = _ids(train), _ids(roll)
        v = C.c_double()
        rc = self.lib.ref_weight_sync(self.h, t.ctypes.data_as(abi.i32p), len(t),
                                      r.ctypes.data_as(abi.i32p), len(r), window,
                                      json.dumps(rollout_plan).encode(), C.byref(v))
        if rc:
            raise RefError(rc, self.lib.ref_last_error().decode())
        return v.value

    def partition_candidates(self, gamma_l, gamma_h, k=8, seed=0x5EED, restarts=16, q=0.0, r=1.0,
                             force_local=False, machine=False):
        out = C.c_void_p()
        rc = self.lib.ref_partition_candidates(self.h, q, r, gamma_l, gamma_h, k, seed, restarts,
                                               int(force_local), int(machine), C.byref(out))
        return self._json(rc, out)


class Oracle:
    """The C restatement (oracle/liboracle.so) on one Problem."""

    def __init__(self, problem):
        self.lib = oracle_lib()
        self.problem = problem
        self.c, self.w, self.k = problem.structs()

    def err(self, rc):
        raise RefError(rc, self.lib.or_last_error().decode())

    def train_space(self, ids, opts=None):
        ids = _ids(ids)
        out = C.c_int64()
        rc = self.lib.or_train_space(C.byref(self.c), C.byref(self.w), ids.ctypes.data_as(abi.i32p),
                                     len(ids), C.byref(opts or abi.default_train_opts()), C.byref(out))
        if rc:
            self.err(rc)
        return out.value

    def constrained_search_raw(self, ids, window, opts=None, lo=0, hi=-1):
        ids = _ids(ids)
        res = abi.gp_train_result()
        devs = np.zeros(max(len(ids), 1), dtype=np.int32)
        rc = self.lib.or_constrained_search(C.byref(self.c), C.byref(self.w), C.byref(self.k),
                                            ids.ctypes.data_as(abi.i32p), len(ids), window,
                                            C.byref(opts or abi.default_train_opts()), lo, hi,
                                            C.byref(res), devs.ctypes.data_as(abi.i32p))
        if rc:
            self.err(rc)
        return res, devs

    def constrained_search(self, ids, window, opts=None, lo=0, hi=-1):
        res, devs = self.constrained_search_raw(ids, window, opts, lo, hi)
        return train_result_dict(res, devs)

    def layout_costs(self, ids, lo, hi, opts=None):
        """per_step of every layout of ranks [lo, hi) (+inf: no memory-feasible option)."""
        ids = _ids(ids)
        out = np.zeros(max(hi - lo, 1), dtype=np.float64)
        rc = self.lib.or_layout_costs(C.byref(self.c), C.byref(self.w), C.byref(self.k),
                                      ids.ctypes.data_as(abi.i32p), len(ids),
                                      C.byref(opts or abi.default_train_opts()), lo, hi,
                                      out.ctypes.data_as(C.POINTER(C.c_double)))
        if rc:
            self.err(rc)
        return out[:hi - lo]

    def layout_costs_tab(self, ids, ranges, opts=None):
        """per_step of the layouts of several [lo, hi) rank ranges, concatenated."""
        ids = _ids(ids)
        lo = np.asarray([a for a, _ in ranges], dtype=np.int64)
        hi = np.asarray([b for _, b in ranges], dtype=np.int64)
        out = np.zeros(max(int((hi - lo).sum()), 1), dtype=np.float64)
        rc = self.lib.or_layout_costs_tab(C.byref(self.c), C.byref(self.w), C.byref(self.k),
                                          ids.ctypes.data_as(abi.i32p), len(ids),
                                          C.byref(opts or abi.default_train_opts()), len(ranges),
                                          lo.ctypes.data_as(C.POINTER(C.c_int64)),
                                          hi.ctypes.data_as(C.POINTER(C.c_int64)),
                                          out.ctypes.data_as(C.POINTER(C.c_double)))
        if rc:
            self.err(rc)
        return out[:int((hi - lo).sum())]

    def constrained_search_tab(self, ids, windows, lo=0, hi=-1, threads=None, dump=False, opts=None):
        """Table-memoised restatement over ranks [lo, hi): {window: (cost, rank)}, feasible,
        layouts (and the per_step dump when asked)."""
        ids = _ids(ids)
        windows = list(windows)
        wa = np.asarray(windows, dtype=np.int32)
        cost = np.zeros(len(windows), dtype=np.float64)
        rank = np.zeros(len(windows), dtype=np.int64)
        feas, lay = C.c_int64(), C.c_int64()
        threads = threads or os.cpu_count() or 1
        buf = None
        if dump:
            total = self.train_space(ids)
            h = total if hi < 0 else min(hi, total)
            buf = np.zeros(max(h - lo, 1), dtype=np.float64)
        rc = self.lib.or_constrained_search_tab(
            C.byref(self.c), C.byref(self.w), C.byref(self.k), ids.ctypes.data_as(abi.i32p), len(ids),
            C.byref(opts or abi.default_train_opts()), wa.ctypes.data_as(abi.i32p), len(windows),
            lo, hi, threads, cost.ctypes.data_as(C.POINTER(C.c_double)),
            rank.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(feas), C.byref(lay),
            buf.ctypes.data_as(C.POINTER(C.c_double)) if dump else None)
        if rc:
            self.err(rc)
        out = {"windows": {w: (float(c), int(r)) for w, c, r in zip(windows, cost, rank)},
               "feasible": feas.value, "layouts": lay.value}
        if dump:
            out["per_step"] = buf
        return out

    def train_candidates_search(self, ids, window):
        ids = _ids(ids)
        res = abi.gp_train_result()
        devs = np.zeros(max(len(ids), 1), dtype=np.int32)
        rc = self.lib.or_train_candidates_search(C.byref(self.c), C.byref(self.w), C.byref(self.k),
                                                 ids.ctypes.data_as(abi.i32p), len(ids), window,
                                                 C.byref(res), devs.ctypes.data_as(abi.i32p))
        if rc:
            self.err(rc)
        return train_result_dict(res, devs)

    def brute_milp(self, configs, caps, B, mean_len):
        arr = (abi.gp_config * max(len(configs), 1))(*configs)
        caps = _ids(caps)
        feas, theta, vec = C.c_int32(), C.c_double(), C.c_int64()
        counts = np.zeros(max(len(configs), 1), dtype=np.int32)
        rc = self.lib.or_brute_milp(arr, len(configs), caps.ctypes.data_as(abi.i32p), len(caps), B,
                                   mean_len, C.byref(feas), C.byref(theta),
                                   counts.ctypes.data_as(abi.i32p), C.byref(vec))
        if rc:
            self.err(rc)
        return {"feasible": bool(feas.value), "theta": theta.value,
                "replica_counts": counts[:len(configs)].tolist(), "vectors": vec.value}

    def exhaustive(self, window):
        out = abi.gp_exhaustive_result()
        ids = np.zeros(self.problem.cluster.n, dtype=np.int32)
        rc = self.lib.or_exhaustive_optimum(C.byref(self.c), C.byref(self.w), C.byref(self.k), window,
                                            C.byref(out), ids.ctypes.data_as(abi.i32p))
        if rc:
            self.err(rc)
        return exhaustive_dict(out, ids)

    def schedule(self, eta=-1, seed=4276115, expand=True, restarts=16, tab_threads=0):
        class SchedOpts(C.Structure):
            _fields_ = [("eta_override", C.c_int32), ("seed", C.c_uint64), ("restarts", C.c_int32),
                        ("expand_window", C.c_int32), ("band_widen_step", C.c_double),
                        ("tab_threads", C.c_int32)]
        o = SchedOpts(eta, seed, restarts, int(expand), 0.05, tab_threads)
        out = C.c_void_p()
        rc = self.lib.or_schedule(C.byref(self.c), C.byref(self.w), C.byref(self.k), C.byref(o),
                                  C.byref(out))
        if rc:
            self.err(rc)
        s = C.cast(out, C.c_char_p).value.decode()
        self.lib.or_free(out)
        return json.loads(s)


def train_result_dict(res, devs):
    """gp_train_result -> the reference JSON shape used by ref_constrained_search."""
    d = {"found": bool(res.found), "layouts": res.layouts, "feasible": res.feasible}
    if res.found:
        d["cost"] = res.cost
        d["rank"] = res.rank
        d["stages"] = [{"devices": devs[s.first:s.first + s.count].tolist(), "tp": s.tp, "dp": s.dp,
                        "layers": s.layers} for s in res.stage[:res.n_stages]]
    return d


def exhaustive_dict(out, ids):
    return {"feasible": bool(out.feasible), "objective": out.objective if out.feasible else None,
            "train_set": ids[:out.n_train].tolist(), "partitions": out.partitions,
            "train_candidates": out.train_candidates, "replica_vectors": out.replica_vectors}


def config_dict(c, n_types):
    return {"type_counts": list(c.type_counts[:n_types]), "tp_per_stage": list(c.tp[:c.n_stages]),
            "throughput": c.throughput}


def oracle_configs(orc, ids, max_stages=4):
    import ctypes as C
    ids = _ids(ids)
    out = (abi.gp_config * 4096)()
    n = C.c_int32()
    rc = orc.lib.or_enumerate_configs(C.byref(orc.c), C.byref(orc.w), C.byref(orc.k),
                                      ids.ctypes.data_as(abi.i32p), len(ids),
                                      C.byref(abi.gp_rollout_opts(max_stages)), out, 4096, C.byref(n))
    if rc:
        orc.err(rc)
    return [out[i] for i in range(n.value)]


def oracle_milp(orc, configs, caps, B, mean_len):
    """Returns (rc, result, entries) of the C restatement of solve_milp."""
    import ctypes as C
    arr = (abi.gp_config * max(len(configs), 1))(*configs)
    caps = _ids(caps)
    res = abi.gp_rollout_result()
    ent = (abi.gp_rollout_entry * max(len(configs), 1))()
    rc = orc.lib.or_solve_milp(arr, len(configs), caps.ctypes.data_as(abi.i32p), len(caps), B,
                               mean_len, C.byref(res), ent)
    return rc, res, [ent[i] for i in range(res.n_entries)] if rc == 0 else []


def oracle_weight_sync(orc, train, roll, etypes, ereps, window):
    import ctypes as C
    t, r, et, er = _ids(train), _ids(roll), _ids(etypes), _ids(ereps)
    v = C.c_double()
    rc = orc.lib.or_weight_sync_cost(C.byref(orc.c), C.byref(orc.w), C.byref(orc.k),
                                     t.ctypes.data_as(abi.i32p), len(t), r.ctypes.data_as(abi.i32p),
                                     len(r), et.ctypes.data_as(abi.i32p), er.ctypes.data_as(abi.i32p),
                                     len(et), window, C.byref(v))
    if rc:
        orc.err(rc)
    return v.value


def oracle_partitions(orc, gamma_l, gamma_h, k=8, seed=0x5EED, restarts=16, force_local=False,
                      machine=False):
    """C restatement of graph_partition_candidates -> [(train, objective, fraction)] or raises."""
    import ctypes as C
    g = abi.gp_gamma(0.0, 1.0, gamma_l, gamma_h)
    o = abi.gp_part_opts(12, restarts, seed, 1e-9, int(force_local), int(machine))
    out = (abi.gp_partition * k)()
    ids = np.zeros(orc.problem.cluster.n * k, dtype=np.int32)
    n = C.c_int32()
    rc = orc.lib.or_partition_candidates(C.byref(orc.c), C.byref(g), C.byref(o), k, out,
                                         ids.ctypes.data_as(abi.i32p), C.byref(n))
    if rc:
        orc.err(rc)
    return [(ids[p.train_offset:p.train_offset + p.train_count].tolist(), p.objective,
             p.compute_fraction) for p in out[:n.value]]
