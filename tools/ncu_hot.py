"""Hottest SASS lines (warp-stall samples) of one kernel in an ncu report:
python tools/ncu_hot.py rep.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "-c", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
secs, cur = [], None
for x in rows:
    if x and x[0] == "Kernel Name":
        cur = {"name": x[1], "rows": []}
        secs.append(cur)
    elif x and x[0] == "Address" and cur is not None:
        cur["h"] = x
    elif cur is not None:
        cur["rows"].append(x)
f = lambda v: float(v) if v not in ("", "-") else 0.0  # noqa: E731
for sec in secs[:1]:
    h, rs = sec["h"], sec["rows"]
    si, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot = sum(f(x[si]) for x in rs)
    print(sec["name"][:80], "samples", tot, "instructions", sum(f(x[ei]) for x in rs))
    idx = sorted(range(len(rs)), key=lambda i: -f(rs[i][si]))[:top]
    for i in sorted(idx):
        print(f"{i:5d} {f(rs[i][si]):6.0f} {100 * f(rs[i][si]) / max(tot, 1):5.1f}% {rs[i][ei]:>8}  {rs[i][1][:90]}")
