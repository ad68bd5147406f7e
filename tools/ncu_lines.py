"""Per-source-line instruction / stall share of one kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
data = []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and r[2] == "-":
        try:
            data.append((int(r[7]), float(r[4] or 0), cur, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data)
tst = sum(d[1] for d in data)
print("total warp instructions", tot)
for e, st, f, line, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * e / tot:5.1f}% inst {100 * st / max(tst, 1):5.1f}% stall {f}:{line:>5} {s}")
