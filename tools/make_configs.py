"""Writes the synthetic C2-C5 inputs of SURVEY.md 8(d) (committed; run once).

Type table from proj/data/clusters/desk_mixed.json (H800, H20) plus a
PCIe-class third type; inter-machine 5 GB/s, cross-type 1.5 GB/s
(PAPER.md:337); workload histogram from proj/data/workloads/math_14b.json.
Machine-pair overrides model an IB-connected pair (25 GB/s) and a degraded
link (3 GB/s). Calibration: explicit {compute 0.4, io 0.6} per type.
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TYPES = {
    "H800": {"name": "H800", "flops_tflops": 756, "hbm_gbps": 2000, "hbm_gb": 80, "price_per_hour": 5.28},
    "H20": {"name": "H20", "flops_tflops": 148, "hbm_gbps": 4000, "hbm_gb": 96, "price_per_hour": 1.85},
    "PCIE": {"name": "PCIE", "flops_tflops": 312, "hbm_gbps": 2039, "hbm_gb": 80, "price_per_hour": 2.5},
}
INTRA = {"H800": 200, "H20": 450, "PCIE": 64}
PREFIX = {"H800": "h800", "H20": "h20", "PCIE": "pcie"}


def cluster(layout, overrides=()):
    types = [t for t, _, _ in layout]
    machines = []
    for t, n_machines, per in layout:
        for i in range(n_machines):
            machines.append({"id": f"{PREFIX[t]}-{i}", "gpu_type": t, "count": per})
    bw = {"intra_machine_gbps": {t: INTRA[t] for t in types}, "inter_machine_gbps": 5}
    if len(types) > 1:
        bw["cross_type_gbps"] = 1.5
    if overrides:
        bw["overrides"] = [{"a": a, "b": b, "gbps": g} for a, b, g in overrides]
    return {"gpu_types": [TYPES[t] for t in types], "machines": machines, "bandwidth": bw}


def workload(params_b, layers, hidden, staleness):
    return {"model": {"params_billion": params_b, "num_layers": layers, "hidden_dim": hidden},
            "batch_rollouts": 64, "prompt_len": 512, "staleness": staleness,
            "length_dist": {"histogram": [[1024, 0.4], [2048, 0.4], [4096, 0.2]]},
            "bytes_per_param_train": 18, "bytes_per_param_infer": 2, "reward_cost_const": 0.0,
            "micro_batches": 8}


def calib(types):
    return {"types": {t: {"compute_efficiency": 0.4, "io_efficiency": 0.6} for t in types},
            "model": {"sync_latency_s": 1.0, "stage_latency_penalty": 0.15, "max_concurrency": 4,
                      "activation_coeff": 4.0, "tp_allreduce_coeff": 4.0, "grad_bytes_per_param": 2.0}}


CONFIGS = {
    "c2_16gpu": (cluster([("H800", 1, 8), ("H20", 1, 8)]), workload(7, 28, 3584, 2)),
    "c3_64gpu": (cluster([("H800", 3, 8), ("H20", 3, 8), ("PCIE", 2, 8)],
                         [("h800-0", "h800-1", 25), ("h20-0", "h20-1", 25), ("h800-2", "pcie-0", 3)]),
                 workload(14, 48, 5120, 1)),
    "c4_256gpu": (cluster([("H800", 12, 8), ("H20", 12, 8), ("PCIE", 8, 8)],
                          [("h800-0", "h800-1", 25), ("h20-0", "h20-1", 25), ("h800-5", "pcie-3", 3)]),
                  workload(32, 64, 5120, 2)),
    "c5_1024gpu": (cluster([("H800", 24, 16), ("H20", 24, 16), ("PCIE", 16, 16)],
                           [("h800-0", "h800-1", 25), ("h20-0", "h20-1", 25), ("h800-7", "pcie-5", 3)]),
                   workload(70, 80, 8192, 2)),
}

# tiny clusters (<= 12 devices) exercise the exact bisection tier (src/partition.cpp:212-222)
CONFIGS["t10_tiny"] = (cluster([("H800", 2, 3), ("H20", 1, 4)]), workload(1.5, 28, 1536, 1))
CONFIGS["t8_tiny"] = (cluster([("H20", 2, 2), ("PCIE", 1, 4)], [("h20-0", "h20-1", 25)]),
                      workload(1.5, 28, 1536, 2))

if __name__ == "__main__":
    for name, (cl, wl) in CONFIGS.items():
        types = [t["name"] for t in cl["gpu_types"]]
        for sub, doc in (("clusters", cl), ("workloads", wl), ("calibration", calib(types))):
            with open(os.path.join(ROOT, "data", sub, name + ".json"), "w") as f:
                json.dump(doc, f, indent=1)
                f.write("\n")
    print("wrote", ", ".join(CONFIGS))
