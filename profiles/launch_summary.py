"""Per-kernel share of the last frame in an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv python bench.py ...`).

  python profiles/launch_summary.py profiles/r01_launches_vN.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    data = rows[hi + 1:]
    starts = [i for i, r in enumerate(data) if "preprocess_kernel" in r[ki]]
    agg, tot = collections.OrderedDict(), 0.0
    for r in data[starts[-1]:]:
        name = r[ki].replace("void ", "").split("(")[0][:60]
        v = float(r[vi].replace(",", ""))
        agg[name] = agg.get(name, 0.0) + v
        tot += v
    for n, v in agg.items():
        print(f"{v / 1e3:8.1f} us {100 * v / tot:5.1f}%  {n}")
    print(f"{tot / 1e3:8.1f} us total (serialised, cold-cache)")


if __name__ == "__main__":
    main(sys.argv[1])
