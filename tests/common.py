"""Shared fixtures: the committed configs (data/) and deterministic train sets."""
from __future__ import annotations

import functools
import json
import os
import random

from paper_2511_00796_b200 import load_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "data")
GOLDEN = os.path.join(ROOT, "tests", "golden")
CONFIGS = ["c1_desk_mixed", "c2_16gpu", "c3_64gpu", "c4_256gpu", "c5_1024gpu"]
ETA = {"c1_desk_mixed": 1, "c2_16gpu": 2, "c3_64gpu": 1, "c4_256gpu": 2, "c5_1024gpu": 2}


def read(sub, name):
    with open(os.path.join(DATA, sub, name + ".json")) as f:
        return f.read()


@functools.lru_cache(maxsize=None)
def problem(name):
    return load_problem(read("clusters", name), read("workloads", name), read("calibration", name))


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def random_train_sets(n_devices, count, seed, min_size=1, max_size=None):
    rng = random.Random(seed)
    max_size = max_size or n_devices - 1
    out = []
    for _ in range(count):
        k = rng.randint(min_size, max_size)
        out.append(sorted(rng.sample(range(n_devices), k)))
    return out


def type_prefix_sets(p, lead, sizes):
    """Type-aligned prefix train sets as run_two_phase probes them (src/scheduler.cpp:175-199)."""
    cl = p.cluster
    order = sorted(range(cl.n), key=lambda d: (cl.device_type[d] != lead, cl.device_type[d], d))
    return [sorted(order[:m]) for m in sizes]
