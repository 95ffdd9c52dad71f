"""Top SASS instructions by executed count / stall samples from an ncu report (source page)."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
hdr = rows[0]
iA, iS, iE, iW = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[iE]), int(r[iW]), r[iA][-5:], r[iS].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
stot = sum(d[1] for d in data)
print("total inst", tot, "samples", stot, "n", len(data))
mode = sys.argv[2] if len(sys.argv) > 2 else "exec"
key = 0 if mode == "exec" else 1
if mode == "dump":
    for d in data:
        print(f"{d[2]} {d[0]:>12d} {d[1]:>7d}  {d[3]}")
else:
    for d in sorted(data, key=lambda d: -d[key])[:int(sys.argv[3]) if len(sys.argv) > 3 else 60]:
        print(f"{d[2]} {d[0]:>12d} {d[1]:>7d}  {d[3]}")
