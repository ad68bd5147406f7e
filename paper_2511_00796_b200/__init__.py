"""B200-native plan-evaluation engine for the arXiv 2511.00796 (AReaL-Hex) scheduler.

The product is libgplan.so (CUDA, sm_100a) behind the C ABI in include/gplan.h;
this package holds its sources (csrc/), the build recipe, the reference-format
input loaders and the Python binding. See DESIGN.md / INTEGRATION.md.
"""
from .inputs import Calibration, Cluster, Problem, Workload, load_problem  # noqa: F401

__all__ = ["Calibration", "Cluster", "Problem", "Workload", "load_problem"]
