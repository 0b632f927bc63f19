"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list.
python tools/launch_table.py launches.csv [last_n_calls_divisor]"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("gsicp::", "").replace("<unnamed>::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        rows.append((name, v))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for n, v in rows:
        tot[n] += v
        cnt[n] += 1
    all_ = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'us/div':>10s} {'share':>6s}")
    for n in sorted(tot, key=lambda x: -tot[x]):
        print(f"{n[:60]:60s} {cnt[n]:8d} {tot[n] / 1e3 / div:10.1f} {100 * tot[n] / all_:5.1f}%")


if __name__ == "__main__":
    main()
