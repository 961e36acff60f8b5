"""Summarise an ncu source page (cuda+sass CSV on stdin) into per-source-line stall/instruction shares."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
cur, hdr, out = None, None, []
for row in rows:
    if len(row) == 2 and row[0] in ("File Path", "File Name"):
        cur = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr) or not row[0]:
        continue
    try:
        s, ins = int(row[4]), int(row[7])
    except ValueError:
        continue
    d = dict(zip(hdr[4:], row[4:]))
    out.append((s, ins, cur, row[0], row[1].strip()[:90], d.get("stall_long_sb", ""), d.get("stall_short_sb", ""),
                d.get("stall_wait", "")))
tot = sum(x[0] for x in out) or 1
ti = sum(x[1] for x in out) or 1
print(f"total stall samples {tot}, warp instructions {ti}")
print(" samp%  inst%  long_sb short_sb   wait  line")
for x in sorted(out, reverse=True)[: int(sys.argv[1]) if len(sys.argv) > 1 else 30]:
    print(f"{100 * x[0] / tot:5.1f} {100 * x[1] / ti:6.1f} {x[5]:>8} {x[6]:>8} {x[7]:>6}  {x[2]}:{x[3]} {x[4]}")
