"""Render a bench.py JSON line as the markdown results table used in
README.md / BASELINE.md:  python tools/bench_table.py bench.json"""
import json
import sys


def f(x, d=1):
    return "—" if x is None else (f"{x:.{d}f}" if x >= 1 else f"{x:.3g}")


def main():
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    rl = d["roofline"]
    cpu = d.get("cpu_baseline") or {}
    print("| config | B200 value | roofline frac | e2e | reference CPU (same config) |")
    print("|---|---|---|---|---|")
    print(f"| c4 BAPG n=m=20000 ({d['config']['precision']}) | {f(d['value'], 2)} it/s | "
          f"{f(rl['frac'], 3)} (chain {f(rl['achieved'])} TFLOP/s) | {f(d['e2e']['value'], 2)} it/s | "
          f"{f(cpu.get('value'))} it/s ({cpu.get('cores')} cores) |")
    for k, v in (d.get("configs") or {}).items():
        if not v or v.get("value") is None:
            continue
        r = v.get("roofline") or {}
        c = v.get("cpu_baseline") or {}
        e = (v.get("e2e") or {}).get("value")
        print(f"| {k} ({v.get('precision', '')}) | {f(v['value'])} {v.get('unit', '')} | "
              f"{f(r.get('frac'), 3)} | {f(e)} | {f(c.get('value'))} {c.get('unit', '')} |")
    print(f"\nclocks: {d['clocks']}")


if __name__ == "__main__":
    main()
