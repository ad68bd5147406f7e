"""Print the SASS of K1-fast's candidate loop (R=3, no dump) from a libgplan build and count
its instructions: from the suffix-record load to the near-minimum test, per unrolled copy.
usage: python tools/k1_loop_sass.py [libgplan.so] [-v]"""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "paper_2511_00796_b200/libgplan.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn = "_ZN2gp19k1_layout_scan_fastILi3ELb0EEEvNS_10TrainSpaceENS_11TrainTablesEPK7double2iNS_9ScanRangeEPNS_7NearMinEPy"
body = out.split("Function : " + fn, 1)[1].split("Function : ", 1)[0]
ins = []
for ln in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
pos = [i for i, (_, t) in enumerate(ins) if t.startswith("POPC")]
for p in pos:
    a = p
    while a > 0 and "LDG.E.128.CONSTANT" not in ins[a][1]:
        a -= 1
    b = p
    while b < len(ins) and not ins[b][1].startswith("DSETP.GTU"):
        b += 1
    seg = ins[a:b + 2]
    print(f"copy at {ins[a][0]:#x}: {len(seg)} instructions in address range (incl. rare-path blocks)")
    if "-v" in sys.argv:
        for addr, t in seg:
            print(f"  {addr:6x}  {t}")
