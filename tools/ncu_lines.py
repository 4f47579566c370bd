"""Per-source-line instruction / stall-sample shares from an ncu source-page
CSV (`ncu -i X --page source --csv --print-source cuda,sass`)."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    f = None
    hdr = None
    agg = []
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        agg.append((f, int(r[0]), r[1], ie, st))
    tot = sum(a[3] for a in agg) or 1
    tst = sum(a[4] for a in agg) or 1
    print(f"total instructions {tot:.4g}, samples {tst:.4g}")
    for f, ln, src, ie, st in sorted(agg, key=lambda a: -a[3])[:top]:
        print(f"{100 * ie / tot:5.1f}% inst {100 * st / tst:5.1f}% stall  "
              f"{f.split('/')[-1]}:{ln}  {src.strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
