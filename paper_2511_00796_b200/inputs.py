"""Host-side input model: the reference's JSON documents -> the engine's SoA structs.

Restates the loaders the hot path depends on (they run once, on the host):
  load_cluster_json      src/cluster.cpp:82-252  (units, link expansion, overrides)
  load_workload_json     src/workload.cpp:14-56,70-99 (LengthDistribution mean)
  load_calibration_json  src/calibration.cpp:71-158 (explicit or fitted efficiencies)
Every floating-point expression keeps the reference's order of operations
(Python floats are IEEE doubles without contraction), so the structs handed to
libgplan.so hold bit-identical values to the reference's ClusterGraph /
WorkloadSpec / Calibration — tests/test_inputs.py pins that against the
reference library itself.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import abi


class InputError(ValueError):
    """ParseError / ValidationError of the reference loaders."""


def _pos(v, path):
    v = float(v)
    if not v > 0:
        raise InputError(f"{path} must be > 0, got {v}")
    return v


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class Cluster:
    type_names: list
    type_flops: np.ndarray
    type_hbm_bw: np.ndarray
    type_hbm_cap: np.ndarray
    type_price: np.ndarray
    machine_names: list
    machine_type: np.ndarray
    device_type: np.ndarray
    device_machine: np.ndarray
    links: np.ndarray  # N x N bytes/s
    _keep: list = field(default_factory=list, repr=False)

    @property
    def n(self) -> int:
        return int(self.device_type.shape[0])

    @property
    def device_flops(self):
        return self.type_flops[self.device_type]

    @property
    def device_hbm_bw(self):
        return self.type_hbm_bw[self.device_type]

    @property
    def device_hbm_cap(self):
        return self.type_hbm_cap[self.device_type]

    def struct(self) -> abi.gp_cluster:
        arrs = [_i32(self.device_type), _i32(self.device_machine), _f64(self.device_flops),
                _f64(self.device_hbm_bw), _f64(self.device_hbm_cap), _f64(self.type_flops),
                _f64(self.type_hbm_bw), _f64(self.type_hbm_cap), _f64(self.links)]
        self._keep.append(arrs)
        p = [a.ctypes.data_as(abi.i32p if a.dtype == np.int32 else abi.f64p) for a in arrs]
        return abi.gp_cluster(self.n, len(self.type_names), len(self.machine_names), *p)


def load_cluster(doc) -> Cluster:
    """load_cluster_json (src/cluster.cpp:82-252)."""
    if isinstance(doc, str):
        doc = json.loads(doc)
    types = doc.get("gpu_types")
    if not isinstance(types, list) or not types:
        raise InputError("gpu_types must be a non-empty array")
    names, fl, bw, cap, price = [], [], [], [], []
    for i, t in enumerate(types):
        p = f"gpu_types[{i}]"
        if t["name"] in names:
            raise InputError(f"duplicate gpu_type '{t['name']}'")
        names.append(t["name"])
        fl.append(_pos(t["flops_tflops"], p + ".flops_tflops") * 1e12)
        bw.append(_pos(t["hbm_gbps"], p + ".hbm_gbps") * 1e9)
        cap.append(_pos(t["hbm_gb"], p + ".hbm_gb") * 1e9)
        price.append(float(t["price_per_hour"]))
    machines = doc.get("machines")
    if not isinstance(machines, list) or not machines:
        raise InputError("machines must be a non-empty array")
    mnames, mtype, dtype, dmach = [], [], [], []
    for i, m in enumerate(machines):
        if m["id"] in mnames:
            raise InputError(f"duplicate machine id '{m['id']}'")
        if m["gpu_type"] not in names:
            raise InputError(f"unknown gpu_type '{m['gpu_type']}'")
        count = int(m["count"])
        if count < 1:
            raise InputError(f"machines[{i}].count must be >= 1")
        t = names.index(m["gpu_type"])
        mnames.append(m["id"])
        mtype.append(t)
        dtype += [t] * count
        dmach += [len(mnames) - 1] * count
    bwdoc = doc["bandwidth"]
    intra_doc = bwdoc["intra_machine_gbps"]
    if isinstance(intra_doc, (int, float)):
        intra = {n: _pos(intra_doc, "bandwidth.intra_machine_gbps") for n in names}
    else:
        intra = {}
        for k, v in intra_doc.items():
            if k not in names:
                raise InputError(f"unknown gpu_type '{k}'")
            intra[k] = _pos(v, "bandwidth.intra_machine_gbps." + k)
        for n in names:
            if n not in intra:
                raise InputError(f"bandwidth.intra_machine_gbps missing entry for type '{n}'")
    inter = _pos(bwdoc["inter_machine_gbps"], "bandwidth.inter_machine_gbps")
    if len(names) > 1:
        cross = _pos(bwdoc["cross_type_gbps"], "bandwidth.cross_type_gbps")
    else:
        cross = float(bwdoc.get("cross_type_gbps", inter))
    M = len(mnames)
    # machine-pair table in bytes/s: gbps * 1e9 exactly as the per-device loop computes it
    mp = np.empty((M, M), dtype=np.float64)
    for a in range(M):
        for b in range(M):
            if a == b:
                mp[a, b] = intra[names[mtype[a]]] * 1e9
            else:
                mp[a, b] = (cross if mtype[a] != mtype[b] else inter) * 1e9
    for i, ov in enumerate(bwdoc.get("overrides", [])):
        p = f"bandwidth.overrides[{i}]"
        if ov["a"] not in mnames or ov["b"] not in mnames:
            raise InputError(p + " references an unknown machine id")
        ia, ib = mnames.index(ov["a"]), mnames.index(ov["b"])
        if ia == ib:
            raise InputError(p + " must name two distinct machines")
        mp[ia, ib] = mp[ib, ia] = _pos(ov["gbps"], p + ".gbps") * 1e9
    dm = np.asarray(dmach, dtype=np.int64)
    links = mp[dm][:, dm].copy()
    np.fill_diagonal(links, 0.0)
    return Cluster(names, _f64(fl), _f64(bw), _f64(cap), _f64(price), mnames, _i32(mtype),
                   _i32(dtype), _i32(dmach), _f64(links))


@dataclass
class Workload:
    model_params_b: float
    num_layers: int
    hidden_dim: int
    batch_rollouts: int
    prompt_len: int
    histogram: list
    mean_len: float
    staleness: int
    bytes_per_param_train: float = 18.0
    bytes_per_param_infer: float = 2.0
    reward_cost_const: float = 0.0
    micro_batches: int = 8

    # inc/workload.hpp:51-58
    def params(self):
        return self.model_params_b * 1e9

    def mean_total_len(self):
        return self.prompt_len + self.mean_len

    def tokens_per_step(self):
        return self.batch_rollouts * self.mean_total_len()

    def model_bytes_infer(self):
        return self.params() * self.bytes_per_param_infer

    def kv_bytes_per_token(self):
        return 4.0 * self.hidden_dim * self.num_layers

    def struct(self) -> abi.gp_workload:
        return abi.gp_workload(self.model_params_b, self.num_layers, self.hidden_dim,
                               self.batch_rollouts, self.prompt_len, self.mean_len,
                               self.bytes_per_param_train, self.bytes_per_param_infer,
                               self.reward_cost_const, self.micro_batches, self.staleness)


def length_mean(hist) -> float:
    """LengthDistribution ctor (src/workload.cpp:14-41): sort, validate, sequential mean."""
    h = sorted((int(l), float(p)) for l, p in hist)
    if not h:
        raise InputError("length distribution must have at least one bucket")
    total = 0.0
    for l, p in h:
        if l <= 0:
            raise InputError("rollout lengths must be positive integers")
        if p < 0:
            raise InputError("length probabilities must be non-negative")
        total += p
    if abs(total - 1.0) > 1e-9:
        raise InputError("length probabilities must sum to 1")
    mean = 0.0
    for l, p in h:
        mean += l * p
    return mean


def load_workload(doc) -> Workload:
    """load_workload_json (src/workload.cpp:71-99)."""
    if isinstance(doc, str):
        doc = json.loads(doc)
    m = doc["model"]
    hist = doc["length_dist"]["histogram"]
    w = Workload(float(m["params_billion"]), int(m["num_layers"]), int(m["hidden_dim"]),
                 int(doc["batch_rollouts"]), int(doc["prompt_len"]), hist, length_mean(hist),
                 int(doc["staleness"]), float(doc.get("bytes_per_param_train", 18.0)),
                 float(doc.get("bytes_per_param_infer", 2.0)), float(doc.get("reward_cost_const", 0.0)),
                 int(doc.get("micro_batches", 8)))
    # WorkloadSpec::validate (src/workload.cpp:58-69)
    if not w.model_params_b > 0 or w.num_layers < 1 or w.hidden_dim < 1 or w.batch_rollouts < 1 \
            or w.prompt_len < 0 or w.staleness < 0 or w.micro_batches < 1:
        raise InputError("invalid workload")
    return w


@dataclass
class Calibration:
    compute_eff: np.ndarray  # by cluster type index
    io_eff: np.ndarray
    sync_latency_s: float = 1.0
    stage_latency_penalty: float = 0.15
    max_concurrency: int = 4
    activation_coeff: float = 4.0
    tp_allreduce_coeff: float = 4.0
    grad_bytes_per_param: float = 2.0
    _keep: list = field(default_factory=list, repr=False)

    def struct(self) -> abi.gp_calib:
        ce, io = _f64(self.compute_eff), _f64(self.io_eff)
        self._keep.append((ce, io))
        return abi.gp_calib(ce.ctypes.data_as(abi.f64p), io.ctypes.data_as(abi.f64p),
                            self.sync_latency_s, self.stage_latency_penalty, self.max_concurrency,
                            self.activation_coeff, self.tp_allreduce_coeff, self.grad_bytes_per_param)


def _trunc_i32_x86(x: float) -> int:
    if not (-2147483649.0 < x < 2147483648.0):
        return -2147483648
    return int(x)


def _single_device_concurrency(cl: Cluster, w: Workload, t: int, max_conc: int) -> int:
    """replica_concurrency (src/cost_model.cpp:128-148) for a 1-device, 1-stage replica."""
    best = max_conc
    layers = w.num_layers  # layers_for_stage(L, 1, 0)
    lf = layers / w.num_layers
    weight = w.params() * lf * w.bytes_per_param_infer / 1
    free = cl.type_hbm_cap[t] - weight
    if free < 0:
        return 0
    kv = w.kv_bytes_per_token() * w.mean_total_len() * lf / 1
    if kv > 0:
        best = min(best, _trunc_i32_x86(free / kv))
    return max(best, 0)


def load_calibration(doc, cl: Cluster, w: Workload) -> Calibration:
    """load_calibration_json / fit_calibration (src/calibration.cpp:71-158)."""
    if doc is None:
        n = len(cl.type_names)  # default_calibration: TypeEfficiency{} per type
        return Calibration(_f64([0.35] * n), _f64([0.6] * n))
    if isinstance(doc, str):
        doc = json.loads(doc)
    m = doc.get("model", {})
    kw = dict(sync_latency_s=float(m.get("sync_latency_s", 1.0)),
              stage_latency_penalty=float(m.get("stage_latency_penalty", 0.15)),
              max_concurrency=int(m.get("max_concurrency", 4)),
              activation_coeff=float(m.get("activation_coeff", 4.0)),
              tp_allreduce_coeff=float(m.get("tp_allreduce_coeff", 4.0)),
              grad_bytes_per_param=float(m.get("grad_bytes_per_param", 2.0)))
    ce, io = [], []
    if "fit_targets" in doc:
        tg = doc["fit_targets"]
        for t, name in enumerate(cl.type_names):
            if name not in tg:
                raise InputError(f"no per-token cost target for gpu_type '{name}'")
            inf = float(tg[name]["per_token_inference_cost"])
            tr = float(tg[name]["per_token_training_cost"])
            price_per_s = cl.type_price[t] / 3600.0
            train_tps = price_per_s / tr
            c_eff = train_tps * (6.0 * w.params()) / cl.type_flops[t]
            conc = _single_device_concurrency(cl, w, t, kw["max_concurrency"])
            if conc < 1:
                raise InputError(f"model does not fit on a single '{name}' device")
            infer_tps = price_per_s / inf
            raw_io = conc * cl.type_hbm_bw[t] / w.model_bytes_infer()
            io_eff = infer_tps / raw_io
            for v in (c_eff, io_eff):
                if not (v > 0) or v > 1.0:
                    raise InputError(f"fitted efficiency for '{name}' outside (0, 1]")
            ce.append(c_eff)
            io.append(io_eff)
    else:
        types = doc["types"]
        for name in cl.type_names:
            if name not in types:
                raise InputError(f"no calibration entry for gpu_type '{name}'")
            ce.append(float(types[name]["compute_efficiency"]))
            io.append(float(types[name]["io_efficiency"]))
    return Calibration(_f64(ce), _f64(io), **kw)


@dataclass
class Problem:
    """One (cluster, workload, calibration) instance as the engine consumes it."""
    cluster: Cluster
    workload: Workload
    calib: Calibration
    texts: tuple = ()

    def structs(self):
        return self.cluster.struct(), self.workload.struct(), self.calib.struct()


def load_problem(cluster_doc, workload_doc, calib_doc=None) -> Problem:
    ctext = cluster_doc if isinstance(cluster_doc, str) else json.dumps(cluster_doc)
    wtext = workload_doc if isinstance(workload_doc, str) else json.dumps(workload_doc)
    ktext = calib_doc if (calib_doc is None or isinstance(calib_doc, str)) else json.dumps(calib_doc)
    cl = load_cluster(ctext)
    w = load_workload(wtext)
    k = load_calibration(ktext, cl, w)
    return Problem(cl, w, k, (ctext, wtext, ktext or ""))
