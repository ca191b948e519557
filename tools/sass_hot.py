"""Summarise an `ncu --page source --csv` SASS dump: top instructions by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
body = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break  # only the first launch of the dump
    if len(r) == len(h):
        body.append(dict(zip(h, r)))
tot = sum(int(b["Warp Stall Sampling (All Samples)"] or 0) for b in body)
print("total samples", tot, "instructions", len(body))
idx = sorted(range(len(body)), key=lambda i: -int(body[i]["Warp Stall Sampling (All Samples)"] or 0))
for i in sorted(idx[:n]):
    b = body[i]
    s = int(b["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{i:5d} {100*s/max(tot,1):5.1f}% exec={b['Instructions Executed']:>8} {b['Source'].strip()[:90]}")
