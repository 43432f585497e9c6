"""Summarise an ncu --page source --print-source sass CSV: totals, stall reasons and hot blocks.

usage: ncu -i X.ncu-rep --page source --csv --print-source sass > x.csv
       python profiles/sass_hotspots.py x.csv [block=40]
"""
import csv
import sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main(path, block=40):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    samp = "Warp Stall Sampling (All Samples)"
    tot = sum(f(d[samp]) for d in data)
    inst = sum(f(d["Instructions Executed"]) for d in data)
    print(f"samples {tot:.0f}  warp-instructions {inst / 1e6:.1f}M")
    stalls = [k for k in hdr if k.startswith("stall_")]
    agg = {k: sum(f(d[k]) for d in data) for k in stalls}
    print("stalls:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for i in range(0, len(data), block):
        s = sum(f(d[samp]) for d in data[i:i + block])
        n = sum(f(d["Instructions Executed"]) for d in data[i:i + block])
        if s > 0.01 * tot:
            mid = data[min(i + block // 2, len(data) - 1)]["Source"][:60]
            print(f"{i:5d}-{i + block - 1:5d} {100 * s / tot:5.1f}% samples {n / 1e6:7.1f}M inst  e.g. {mid}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
