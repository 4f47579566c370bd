"""Summarise an `ncu --metrics … --csv` launch list: one block per launch
with the metric values (used for the profiles/ text summaries)."""
import csv
import sys


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = {}
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        if key not in launches:
            launches[key] = {"kernel": d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")}
            order.append(key)
        launches[key][d["Metric Name"]] = f'{d["Metric Value"]} {d.get("Metric Unit", "")}'.strip()
    print(title)
    print("(ncu --clock-control none; per-launch times are cold-cache and serialised)")
    for k in order:
        L = launches[k]
        print("-" * 100)
        print(f'{"Kernel":<60} {L.pop("kernel")}')
        for m in sorted(L):
            print(f"{m:<60} {L[m]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
