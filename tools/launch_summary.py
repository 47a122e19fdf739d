"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count,
total and mean device time, share.  Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
tot = collections.Counter()
cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0]
    tot[name] += float(r[-1])
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total_ms':>10s} {'mean_us':>10s} {'share':>7s}")
for k, v in tot.most_common():
    print(f"{k[:40]:40s} {cnt[k]:8d} {v / 1e6:10.3f} {v / cnt[k] / 1e3:10.2f} {v / T * 100:6.1f}%")
print(f"{'total':40s} {sum(cnt.values()):8d} {T / 1e6:10.3f}")
