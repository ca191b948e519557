"""Per-kernel timeline of the SPrM pre-pass train step (CUPTI via
torch.profiler): for every kernel of the step, its average start offset from
the step's first kernel and its average duration, over the middle steps of a
pre-pass; plus the average step period. Usage:
  python tools/sprm_timeline.py [N_BYTES] -> gpurun_out/sprm_timeline.json"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
raw = P.synth("genome", n, 5, 10)
cfg = P.CompressConfig(workers=2, selector_threshold=0)
def run():
    try:
        P.compress(raw, cfg)
    except P.PmklcError as e:  # timing experiments that break the model still time the pre-pass
        print("compress:", e)


run()  # warm
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
trace = out / "sprm_trace.json"
prof.export_chrome_trace(str(trace))
ev = [e for e in json.load(open(trace))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
name = lambda e: e["name"].replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0]
starts = [e["ts"] for e in ev if "k_sprm_prep" in name(e)]
steps = len(starts)
lo, hi = steps // 4, 3 * steps // 4  # middle half of the pre-pass
per = defaultdict(lambda: [0.0, 0.0, 0])
for i in range(lo, hi):
    a, b = starts[i], starts[i + 1]
    seen = defaultdict(int)
    for e in ev:
        if a <= e["ts"] < b:
            k = name(e)
            seen[k] += 1
            key = f"{k}#{seen[k]}" if seen[k] > 1 else k
            per[key][0] += e["ts"] - a
            per[key][1] += e["dur"]
            per[key][2] += 1
period = (starts[hi] - starts[lo]) / (hi - lo)
rows = sorted(((k, v[0] / v[2], v[1] / v[2]) for k, v in per.items()), key=lambda r: r[1])
res = {"steps": steps, "period_us": period,
       "kernels": [{"kernel": k, "start_us": round(s, 2), "dur_us": round(d, 2), "end_us": round(s + d, 2)}
                   for k, s, d in rows]}
json.dump(res, open(out / "sprm_timeline.json", "w"), indent=1)
print(f"step period {period:.1f} us over {hi - lo} steps")
for k, s, d in rows:
    print(f"  {s:7.1f} +{d:6.1f} -> {s + d:7.1f}  {k}")
