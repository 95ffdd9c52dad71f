"""Turn a round's gpurun_out/ evidence into committed summaries under profiles/.

    python scripts/summarize_profiles.py <round-tag>      e.g. r01

Reads gpurun_out/launches.csv (ncu launch list of the bench command), gpurun_out/prof_exact.ncu-rep
and prof_fp32.ncu-rep (ncu --set full of the hot kernel) and writes:
  profiles/<tag>_launches.txt        per-kernel launch times and share of the dose step
  profiles/<tag>_ncu_<family>.txt    key throughput / memory / stall metrics + hottest SASS lines
  profiles/dram_bytes_per_launch.json  DRAM read+write bytes per launch (bench.py "traffic")
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("DG_PROFILES_OUT", os.path.join(ROOT, "profiles"))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def launches(tag):
    path = os.path.join(OUT, "launches.csv")
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            name = d["Kernel Name"].split("(")[0]
            v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else
                                            1.0 if d["Metric Unit"] == "us" else 1e3)
            per.setdefault(name, []).append(v)
    dose = {k: v for k, v in per.items() if "gen_" not in k and "cub::" not in k and
            "row_extents" not in k and "split_rows" not in k and "validate" not in k and
            "build_" not in k}

    def family(k):  # the bench runs the exact family, then the fp32 side line
        return "fp32" if ("float" in k or "f32" in k) else "exact"  # k_x_to_f32: fp32 x staging

    # one dose of a family = the sum of its kernels' average launch times
    step = collections.defaultdict(float)
    for k, v in dose.items():
        step[family(k)] += sum(v) / len(v)
    lines = [f"# {tag}: ncu launch list of `python bench.py --steps 3 --warmup 3` (C2, exact "
             "family then the fp32 side line), gpu__time_duration.sum, --clock-control none "
             "(cold-cache, serialised launches); share = avg launch time / the family's dose",
             f"{'kernel':70s} {'launches':>8s} {'avg us':>10s} {'share of dose':>14s}"]
    for k, v in per.items():
        avg = sum(v) / len(v)
        share = avg / step[family(k)] if k in dose else float("nan")
        lines.append(f"{k[:70]:70s} {len(v):8d} {avg:10.1f} {share:14.3f}")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def ncu(tag, family):
    rep = os.path.join(OUT, f"prof_{family}.ncu-rep")
    if not os.path.exists(rep):
        return None
    summ = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                          capture_output=True, text=True).stdout
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_sass_hot.py"), rep,
                          "stall", "25"], capture_output=True, text=True).stdout
    cfg = "C4" if family == "c4" else "C2"
    text = (f"# {tag}: ncu --set full --clock-control none, dose kernels k_slices / k_tiles (+ k_dense) ({cfg}, {family})\n"
            + summ + "\n# hottest SASS by warp-stall samples (addr, executed, samples, instr)\n" + hot)
    open(os.path.join(PROF, f"{tag}_ncu_{family}.txt"), "w").write(text)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    hdr, units = r[0], r[1]

    def get(vals, k):
        v = float(vals[hdr.index(k)])
        u = units[hdr.index(k)]
        return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1)

    # one dose's kernels (k_tiles, and k_dense when the plan uses it): DRAM bytes of the first
    # capture of each kernel, keyed like bench.py's roofline.kernels names
    out = {}
    for v in r[2:]:
        name = v[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""
        key = ("dense_values" if "k_dense_values" in name else "dense" if "k_dense" in name else
               "slices" if "k_slices" in name else "tiles")
        if key not in out:
            out[key] = get(v, "dram__bytes_read.sum") + get(v, "dram__bytes_write.sum")
    return out


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        launches(tag)
    tf = os.path.join(PROF, "dram_bytes_per_launch.json")
    traffic = json.load(open(tf)) if os.path.exists(tf) else {}
    # keys: <config>:<accumulation>:<kernel name in dg_kernel_times> (read by bench.py)
    for fam, prefix, tiles in (("exact", "c2:exact", "tiles[w0]"), ("fp32", "c2:fp32", "tiles[w0]"),
                               ("c4", "c4:exact", "tiles[fused]")):
        t = ncu(tag, fam)
        if t is None:
            continue
        for k, b in t.items():  # slices: bench.py looks the name up without its "[...]" suffix
            traffic[f"{prefix}:{tiles if k == 'tiles' else k}"] = int(b)
            print(fam, k, "dram bytes per launch", b)
    json.dump(traffic, open(tf, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
