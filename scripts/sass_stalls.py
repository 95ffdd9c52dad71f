"""Per-instruction stall breakdown of an ncu source page (--page source --csv --print-source sass):
    python scripts/sass_stalls.py <sass.csv> [top] [kernel-name substring]
Prints stall totals by reason and the hottest instructions with their dominant stall (the last
kernel section whose name matches, when the page holds several)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = sys.argv[3] if len(sys.argv) > 3 else ""
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1] if len(r) > 1 else "", "rows": []}
        sections.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sec = [x for x in sections if want in x["name"]][-1]
print("#", sec["name"][:100])
hdr = sec["rows"][0]
data = [dict(zip(hdr, r)) for r in sec["rows"][1:] if len(r) == len(hdr)]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: sum(float(d[r] or 0) for d in data) for r in reasons}
allsamp = sum(tot.values())
print("samples", allsamp, "instructions executed", sum(float(d["Instructions Executed"] or 0) for d in data))
for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {r:28s} {v:10.0f} {100 * v / allsamp:5.1f}%")
hot = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:top]
for d in hot:
    st = max(reasons, key=lambda r: float(d[r] or 0))
    print(f"{d['Address'][-5:]} {int(float(d['Instructions Executed'] or 0)):10d} "
          f"{d['Warp Stall Sampling (All Samples)']:>7s} {st[6:]:14s} {d['Source'].strip()[:70]}")
