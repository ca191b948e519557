"""Concurrent kernel timeline of one compress (CUPTI via torch.profiler):
per-stream busy time and the main stream's idle gaps over the plateau ticks.
Usage: python tools/timeline.py N_BYTES W [spum] -> gpurun_out/timeline.json"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 128
spum = len(sys.argv) > 3 and sys.argv[3] == "spum"
raw = P.synth("markov3", n, 12345)
cfg = P.CompressConfig(workers=w)
if spum:
    P.write_bigru("/tmp/tl_spum.bin", 3, 32, 4, 0xACE3)
    cfg.pub_model_path = "/tmp/tl_spum.bin"
P.compress(raw, cfg)  # warm (graphs, pools)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    P.compress(raw, cfg)
    torch.cuda.synchronize()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "timeline_trace.json"))
ev = [e for e in json.load(open(out / "timeline_trace.json"))["traceEvents"]
      if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
# plateau window: the middle half of the run
a, b = t0 + 0.25 * (t1 - t0), t0 + 0.75 * (t1 - t0)
busy = defaultdict(float)
per_kernel = defaultdict(lambda: defaultdict(float))
for e in ev:
    s, f = max(e["ts"], a), min(e["ts"] + e["dur"], b)
    if f > s:
        st = e["args"].get("stream", -1)
        busy[st] += f - s
        nm = e["name"].replace("(anonymous namespace)::", "").replace("void ", "")
        per_kernel[st][nm.split("(")[0].split("<")[0].split("::")[-1]] += f - s
# union of all streams' kernels (device busy) in the window
iv = sorted((max(e["ts"], a), min(e["ts"] + e["dur"], b)) for e in ev if min(e["ts"] + e["dur"], b) > max(e["ts"], a))
union, cs, ce = 0.0, None, None
for s, f in iv:
    if cs is None or s > ce:
        if cs is not None:
            union += ce - cs
        cs, ce = s, f
    else:
        ce = max(ce, f)
if cs is not None:
    union += ce - cs
win = b - a
res = {"window_us": win, "device_busy_frac": union / win,
       "streams": {str(k): {"busy_frac": v / win,
                            "top": sorted(((n_, round(t / win, 4)) for n_, t in per_kernel[k].items()),
                                          key=lambda x: -x[1])[:8]}
                   for k, v in sorted(busy.items(), key=lambda kv: -kv[1])}}
json.dump(res, open(out / "timeline.json", "w"), indent=1)
for k, v in res["streams"].items():
    print(f"stream {k}: busy {v['busy_frac']:.3f}  " + ", ".join(f"{n_} {t:.3f}" for n_, t in v["top"]))
print(f"device busy {res['device_busy_frac']:.3f} over {win/1e3:.1f} ms")
