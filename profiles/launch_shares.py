"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python profiles/launch_shares.py profiles/r1_launches.csv "<command line>" > profiles/r1_launch_shares.txt
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        v = float(r[vi].replace(",", ""))
        tot[r[ki]] += v
        cnt[r[ki]] += 1
T = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print("share   launches  total_ns  kernel")
for k, v in tot.most_common():
    print(f"{100 * v / T:6.2f}%  {cnt[k]:4d}  {v:12.0f}  {k[:90]}")
