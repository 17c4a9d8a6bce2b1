"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv):
usage: launch_summary.py launches.csv -> kernel, launches, total us, mean us, share of all launches."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = r[4].split("(")[0].replace("kur::<unnamed>::", "")
        t = float(r[14]) / (1e3 if r[13] == "ns" else 1.0)
        tot[name][0] += 1
        tot[name][1] += t
    all_us = sum(v[1] for v in tot.values())
    print(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share':>7s}")
    for k, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:8d} {t:12.1f} {t / n:10.2f} {t / all_us:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
