"""Summarise an `ncu --page source --csv` SASS dump: top instructions by stall
samples with their dominant stall reasons, and total warp-instructions."""
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
num = lambda v: float(v.replace(",", "")) if v and v.replace(",", "").replace(".", "").isdigit() else 0.0
tot = sum(num(b["Warp Stall Sampling (All Samples)"]) for b in body)
ins = sum(num(b["Instructions Executed"]) for b in body)
print(f"total samples {tot:.0f}, instructions {len(body)}, warp-instructions executed {ins:.0f}")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(num(b[k]) for b in body) for k in reasons}
at = sum(agg.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {100*v/at:.0f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
idx = sorted(range(len(body)), key=lambda i: -num(body[i]["Warp Stall Sampling (All Samples)"]))
for i in sorted(idx[:n]):
    b = body[i]
    s = num(b["Warp Stall Sampling (All Samples)"])
    top = sorted(((num(b[k]), k[6:]) for k in reasons), reverse=True)[:2]
    why = " ".join(f"{k}:{v:.0f}" for v, k in top if v)
    print(f"{i:5d} {100*s/max(tot,1):5.1f}% exec={b['Instructions Executed']:>8} {b['Source'].strip()[:70]:70s} {why}")
