"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch).

    python tools/launch_table.py launches.csv [--skip N]
"""
import csv
import sys

path = sys.argv[1]
skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
        if r["Metric Name"] == "gpu__time_duration.sum"][skip:]
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
tot = 0.0
for r in rows:
    ms = float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
    tot += ms
    print(f'{r["Kernel Name"][:70]:70s} {r["Grid Size"]:>14s} {ms:9.3f} ms')
print(f"{len(rows)} launches, {tot:.3f} ms")
