"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)
        name = r["Kernel Name"].split("(")[0]
        rows.append((name, us))
    tot = sum(u for _, u in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for n, u in rows:
        agg[n][0] += 1
        agg[n][1] += u
    lines = [f"launches {len(rows)} total us {tot:.1f}"]
    for n, (c, u) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{n[:40]:40s} n={c:5d} total={u:11.1f}us avg={u / c:9.2f}us {100 * u / tot:5.1f}%")
    s = "\n".join(lines)
    print(s)
    if out:
        open(out, "w").write(s + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
