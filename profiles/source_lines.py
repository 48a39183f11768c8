"""Per-CUDA-source-line instruction and stall-sample shares of one kernel in an
ncu report (`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`).

  python profiles/source_lines.py X.ncu-rep [kernel-regex] [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kernel=None, top=40):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        cmd += ["-k", "regex:" + kernel]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, agg = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr = r
        elif hdr and r and r[0].isdigit() and len(r) == len(hdr):
            ii = hdr.index("Instructions Executed")
            si = hdr.index("Warp Stall Sampling (All Samples)")
            f = lambda x: float(x) if x not in ("", "-") else 0.0
            agg.append((cur, int(r[0]), r[1].strip(), f(r[ii]), f(r[si])))
    ti = sum(a[3] for a in agg) or 1
    ts = sum(a[4] for a in agg) or 1
    print(f"total warp instructions {ti:.3e}, samples {ts:.0f}")
    for a in sorted(agg, key=lambda a: -a[3])[:top]:
        print(f"{100 * a[3] / ti:5.1f}% inst {100 * a[4] / ts:5.1f}% smp  {a[0]}:{a[1]}  {a[2][:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, int(sys.argv[3]) if len(sys.argv) > 3 else 40)
