"""Split a K1-fast ncu report's executed warp instructions into the per-candidate loop and the
per-prefix (table build) part by source line ranges of train.cu (the candidate loop lines are
passed as lo-hi), and report warp-instructions per candidate for each."""
import csv
import io
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cands = float(sys.argv[4]) if len(sys.argv) > 4 else 2415919104
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None
loop = pref = 0
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Function Name", "Line No") or not r[0] or r[2] != "-":
        continue
    try:
        line, e = int(r[0]), int(r[7])
    except ValueError:
        continue
    if cur == "train.cu" and lo <= line <= hi:
        loop += e
    else:
        pref += e
print(f"loop {loop / cands:.3f}  rest {pref / cands:.3f}  total {(loop + pref) / cands:.3f} warp-inst/candidate")
