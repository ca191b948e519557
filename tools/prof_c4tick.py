"""Kernel breakdown of the config-4 tick regime (flags 6: SPrM + DM, W=256
blocks, ~20 chunks in flight under the SMP stagger) on a smaller input:
decompress of a 40 MB flags-6 container (no pre-pass in the decoder), CUPTI
via torch.profiler. Per kernel: launches, total and average device time,
and the share of the decode's wall time.
Usage: python tools/prof_c4tick.py [N_BYTES] [W] -> gpurun_out/c4tick.json"""
import json
import sys
import time
from collections import defaultdict
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2507_12805_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
w = int(sys.argv[2]) if len(sys.argv) > 2 else 256
spum = len(sys.argv) > 3 and sys.argv[3] == "spum"  # config-3 models (SPuM + DM, flags 5)
if spum:
    import tempfile
    raw = P.synth("genome", n, 2025, 10)
    pub = str(Path(tempfile.mkdtemp()) / "spum.bin")
    P.write_bigru(pub, 3, 32, 4, 0xACE3, layers=2)
    cfg = P.CompressConfig(workers=w, pub_model_path=pub)
else:
    pub = ""
    raw = P.synth("genome", n, 2026, 10)
    cfg = P.CompressConfig(workers=w, selector_threshold=0)
blob = P.compress(raw, cfg)
assert blob[5] == (5 if spum else 6), blob[5]
P.decompress(blob, pub)  # warm
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    out_b = P.decompress(blob, pub)
    torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e6
assert out_b == raw
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace("/tmp/c4tick_trace.json")
ev = [e for e in json.load(open("/tmp/c4tick_trace.json"))["traceEvents"] if e.get("cat") == "kernel"]
name = lambda e: e["name"].replace("(anonymous namespace)::", "").replace("void ", "").replace("pmklc_b200::", "").split("(")[0]
agg = defaultdict(lambda: [0, 0.0])
streams = defaultdict(float)
for e in ev:
    agg[name(e)][0] += 1
    agg[name(e)][1] += e["dur"]
    streams[e.get("tid")] += e["dur"]
ticks = agg.get("k_tick_advance", [1])[0]
span = max(e["ts"] + e["dur"] for e in ev) - min(e["ts"] for e in ev)
rows = sorted(agg.items(), key=lambda kv: -kv[1][1])
res = {"bytes": n, "workers": w, "ticks": ticks, "span_us": span, "wall_us": wall,
       "us_per_tick": span / max(ticks, 1),
       "streams_busy_us": {str(k): v for k, v in streams.items()},
       "kernels": [{"kernel": k, "n": c, "total_us": round(t, 1), "avg_us": round(t / c, 2),
                    "per_tick_us": round(t / max(ticks, 1), 2)} for k, (c, t) in rows]}
json.dump(res, open(out / "c4tick.json", "w"), indent=1)
print(f"decode {n} B W={w}: {ticks} ticks, span {span / 1e3:.1f} ms, {span / max(ticks, 1):.1f} us/tick")
print("stream busy (us):", {k: round(v) for k, v in streams.items()})
for k, (c, t) in rows[:30]:
    print(f"  {t / 1e3:9.1f} ms  n={c:6d}  avg {t / c:8.1f} us  per-tick {t / max(ticks, 1):7.1f} us  {k}")

# one plateau tick: every kernel's stream, start and end relative to the tick's k_tick_advance
adv = sorted(e["ts"] for e in ev if name(e) == "k_tick_advance")
if len(adv) > 10:
    i = len(adv) // 2
    a, b = adv[i], adv[i + 1]
    tick = sorted((e for e in ev if a <= e["ts"] < b), key=lambda e: e["ts"])
    res["plateau_tick"] = [{"kernel": name(e), "stream": e.get("tid"), "start_us": round(e["ts"] - a, 1),
                            "dur_us": round(e["dur"], 1)} for e in tick]
    json.dump(res, open(out / "c4tick.json", "w"), indent=1)
    print(f"plateau tick {i}: {b - a:.1f} us")
    for k in res["plateau_tick"]:
        print(f"  s{k['stream']:>3} {k['start_us']:8.1f} +{k['dur_us']:7.1f}  {k['kernel']}")
