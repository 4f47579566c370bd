"""Per-SASS-instruction stall breakdown from an ncu source-page CSV
(`ncu -i X --page source --csv --print-source cuda,sass`): the top
instructions by one stall reason, with the CUDA line they belong to.

    python tools/ncu_sass_stalls.py src.csv [stall_long_sb] [top]
"""
import csv
import sys


def main(path, reason="stall_long_sb", top=25):
    rows = list(csv.reader(open(path, encoding="utf-8", errors="replace")))
    hdr, line, src = None, None, ""
    out, tot = [], {}
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0].isdigit():
            line, src = int(r[0]), r[1]
            continue
        d = dict(zip(hdr, r))
        try:
            v = float(d.get(reason) or 0)
        except ValueError:
            continue
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    tot[k] = tot.get(k, 0.0) + float(d.get(k) or 0)
                except ValueError:
                    pass
        out.append((v, line, r[3].strip(), src.strip()[:60]))
    out.sort(reverse=True)
    s = sum(tot.values()) or 1
    print("stall totals:", ", ".join(f"{k[6:]} {v / s:.1%}" for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
    for v, ln, sass, c in out[:top]:
        print(f"{v:8.0f}  L{ln:<5} {sass[:48]:48s} | {c}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb",
         int(sys.argv[3]) if len(sys.argv) > 3 else 25)
