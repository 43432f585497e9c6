"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys


def summarise(path, frames=1):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = [r for r in csv.DictReader(lines[start:]) if r["Metric Name"] == "gpu__time_duration.sum"]
    agg, cnt = {}, {}
    for r in rows:
        n = r["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0]
        scale = 1e-3 if r["Metric Unit"] == "ns" else (1.0 if r["Metric Unit"] == "us" else 1e3)
        agg[n] = agg.get(n, 0.0) + float(r["Metric Value"].replace(",", "")) * scale
        cnt[n] = cnt.get(n, 0) + 1
    tot = sum(agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v / frames:10.1f} us/frame {100 * v / tot:5.1f}%  x{cnt[k] // frames:<3d} {k}")
    print(f"{tot / frames:10.1f} us/frame total, {len(rows) // frames} launches/frame")


if __name__ == "__main__":
    summarise(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)
