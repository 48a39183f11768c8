"""Per-kernel share of the last frame in an ncu launch list
(`ncu --metrics gpu__time_duration.sum[,smsp__inst_executed.sum] --csv --log-file X.csv ...`).

  python profiles/launch_summary.py profiles/r02_launches_render_v2.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    idi = h.index("ID") if "ID" in h else None
    data = rows[hi + 1:]
    t = [r for r in data if mi is None or r[mi] == "gpu__time_duration.sum"]
    ins = {r[idi]: float(r[vi].replace(",", "")) for r in data
           if mi is not None and r[mi] == "smsp__inst_executed.sum"}
    starts = [i for i, r in enumerate(t) if "preprocess_kernel" in r[ki]]
    agg, tot = collections.OrderedDict(), 0.0
    for r in t[starts[-1]:]:
        name = r[ki].replace("void ", "").split("(")[0][:56]
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0.0, 0, 0.0])
        a[0] += v
        a[1] += 1
        a[2] += ins.get(r[idi], 0.0) if idi is not None else 0.0
        tot += v
    for n, (v, c, i) in agg.items():
        print(f"{v / 1e3:8.1f} us {100 * v / tot:5.1f}%  x{c:<2d} {i / 1e6:7.1f}M inst  {n}")
    print(f"{tot / 1e3:8.1f} us total (serialised, cold-cache)")


if __name__ == "__main__":
    main(sys.argv[1])
