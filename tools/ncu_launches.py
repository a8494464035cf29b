"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram__bytes_read/write.sum]) by kernel.

usage: ncu_launches.py CSV [top] [--last-matvec]
Per kernel: launches, total ms, and DRAM GB when captured.  --last-matvec prints the launches of the final
matvec (from the last gather_rows launch to the end) with per-launch time, DRAM bytes and share."""
import csv
import sys
from collections import OrderedDict, defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iid, ik, im, iv, iu = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
launch = OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[iv].replace(",", ""))
    except ValueError:
        continue
    u = r[iu]
    if r[im] == "gpu__time_duration.sum":
        v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(u, 1.0)
        key = "ms"
    else:
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        key = "bytes"
    d = launch.setdefault(r[iid], {"name": r[ik].split("(")[0].replace("void ", "")[:60], "ms": 0.0, "bytes": 0.0})
    d[key] += v
agg = defaultdict(lambda: [0, 0.0, 0.0])
for d in launch.values():
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d["ms"]
    a[2] += d["bytes"]
top = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
print("launches %d, total %.2f ms" % (len(launch), sum(d["ms"] for d in launch.values())))
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print("%-60s n=%5d %10.3f ms %8.2f GB" % (k, n, t, b / 1e9))
if "--last-matvec" in sys.argv:
    seq = list(launch.values())
    start = max(i for i, d in enumerate(seq) if "gather_rows" in d["name"])
    end = next((i + 1 for i in range(start, len(seq)) if "l2p" in seq[i]["name"] or "down_compact<1, 1, 1>" in
                seq[i]["name"] or "down_compact<8, 1, 1>" in seq[i]["name"]), len(seq))
    last = seq[start:end]
    tot = sum(d["ms"] for d in last)
    print("\nlast matvec: %d launches, %.3f ms" % (len(last), tot))
    for d in last:
        gbs = d["bytes"] / (d["ms"] * 1e-3) / 1e9 if d["ms"] else 0.0
        print("  %-58s %8.1f us %8.1f MB %7.0f GB/s %5.1f%%" % (d["name"], d["ms"] * 1e3, d["bytes"] / 1e6, gbs,
                                                            100 * d["ms"] / tot))
