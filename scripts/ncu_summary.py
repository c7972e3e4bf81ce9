"""Summarise ncu outputs into markdown for profiles/.

    python scripts/ncu_summary.py launches <launches.csv>          # kernel share of the run
    python scripts/ncu_summary.py full <report.ncu-rep> [--id N]   # key metrics + stall reasons
"""
import collections
import csv
import io
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    for d in data:
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0][:60]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | mean us | total us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Achieved Active Warps Per SM",
        "Theoretical Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Grid Size",
        "Block Size", "Cluster Size", "Issue Slots Busy", "Executed Instructions", "SM Frequency"]


def full(path, kid="0"):
    out = subprocess.run([NCU, "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h = r[0]
    rows = [dict(zip(h, x)) for x in r[1:] if len(x) >= 15]
    kname = next((d["Kernel Name"] for d in rows if d["ID"] == kid), "?")
    print(f"kernel: `{kname[:100]}`\n")
    print("| metric | value |")
    print("|---|---|")
    for d in rows:
        if d["ID"] == kid and d["Metric Name"] in WANT:
            print(f"| {d['Metric Name']} | {d['Metric Value']} {d['Metric Unit']} |")
    raw = subprocess.run([NCU, "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh, units = rr[0], rr[1]
        for x in rr[2:]:
            d = dict(zip(hh, x))
            if d.get("ID") != kid:
                continue
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
            ur = units[hh.index("dram__bytes_read.sum")] if "dram__bytes_read.sum" in hh else ""
            uw = units[hh.index("dram__bytes_write.sum")] if "dram__bytes_write.sum" in hh else ""
            print(f"| dram__bytes_read.sum + write.sum | {rd:.4g} {ur} + {wr:.4g} {uw} |")
    src = subprocess.run([NCU, "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    sr = list(csv.reader(io.StringIO(src)))
    hi = next((i for i, x in enumerate(sr) if x and x[0] == "Address"), None)
    if hi is not None:
        hh = sr[hi]
        stall = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
        tot = collections.Counter()
        for x in sr[hi + 1:]:
            if len(x) != len(hh):
                continue
            d = dict(zip(hh, x))
            for c in stall:
                try:
                    tot[c] += float(d[c] or 0)
                except ValueError:
                    pass
        S = sum(tot.values()) or 1
        print("\nwarp stall samples (share): " + ", ".join(f"{c[6:]} {100 * v / S:.0f}%" for c, v in tot.most_common(8)))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[4] if len(sys.argv) > 4 else "0")
