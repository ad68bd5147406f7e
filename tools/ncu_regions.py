"""Per-region SASS breakdown of one kernel in an ncu report (runs of equal exec count)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
iA, iS, iE = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
data = [(int(r[iA], 16), r[iS].strip(), int(r[iE])) for r in rows[2:] if r[iE].isdigit()]
base = data[0][0]
tot = sum(e for _, _, e in data)
ref = max(e for a, s, e in data if "RCP64H" in s) if any("RCP64H" in s for _, s, _ in data) else 1
groups = []
for a, s, e in data:
    if groups and groups[-1][2] == e:
        groups[-1][1] = a
        groups[-1][3] += 1
        groups[-1][4].append(s)
    else:
        groups.append([a, a, e, 1, [s]])
for g in groups:
    if g[2] * g[3] > tot * 0.004:
        ops = collections.Counter()
        for s in g[4]:
            t = s.split()
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += 1
        print(f"{g[0]-base:6x}-{g[1]-base:6x} x{g[2]/ref:6.3f} n={g[3]:4d} {100*g[2]*g[3]/tot:5.1f}%  "
              + " ".join(f"{k}:{v}" for k, v in ops.most_common(8)))
print(f"warp-inst per RCP64H execution: {tot/ref:.1f}")
