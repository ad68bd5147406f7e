import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from common import problem
from paper_2511_00796_b200 import abi
from paper_2511_00796_b200.engine import Engine, BandInfeasibleError
name = sys.argv[1] if len(sys.argv) > 1 else "c3_64gpu"
p = problem(name)
e = Engine(p)
o = abi.gp_part_opts(12, 16, 4276115, 1e-9, 0, 0)
try:
    e.partition_candidates(0.4, 0.6, 8, o)
except BandInfeasibleError:
    pass
for p16 in [1, 4, 8, 12, 15]:
    g = p16 / 16
    t = time.perf_counter()
    try:
        r = e.partition_candidates(g, g, 8, o); n = len(r)
    except BandInfeasibleError:
        n = -1
    print(name, g, f"{1e3*(time.perf_counter()-t):.2f} ms", n)
