"""Per-source-line stall samples and executed warp-instructions from an ncu report.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
       python profiles/line_hotspots.py x.csv [top=40]
Source-line rows carry the line's totals (inlined code is attributed to the
header line it comes from, so helper lines aggregate every call site).
"""
import csv
import sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    fname, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0] not in ("", "Function Name") and len(r) >= len(hdr):
            d = dict(zip(hdr[2:], r[2:]))
            out.append((f(r[4]), f(r[7]), f"{fname}:{r[0]}", r[1].strip()[:90]))
    tot_s = sum(o[0] for o in out)
    tot_i = sum(o[1] for o in out)
    print(f"samples {tot_s:.0f}, warp-instructions {tot_i / 1e6:.1f}M")
    for s, i, loc, src in sorted(out, key=lambda o: -o[0])[:top]:
        print(f"{100 * s / tot_s:5.1f}% {i / 1e6:7.2f}M  {loc:24s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
