"""Checks bench.py's reference-arm extrapolation against a stock run at the
full chunk geometry, on the same host: the reference compress()+decompress()
of the config-3 prefix holding exactly C chunks of the 100 MB workload's
geometry (W=C, bs=320, L=813: the first C chunks of the bench container),
timed in full, versus the extrapolation from the bounded (32+S)-step samples
to that same workload. Prints one JSON line. Never loads the product library.
Usage: python tools/validate_ref_extrapolation.py [C]"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else min(os.cpu_count() or 1, 16)
O, R, kind = bench.checker()
tmp = tempfile.mkdtemp()
spum = str(Path(tmp) / "spum.bin")
O.write_spum(spum, 3, 32, 4, bench.SPUM_SEED)
full = R.synth("genome", 100_000_000, 2025, 10)
m_chunk = 260417  # the 100 MB plan's first chunks (33,333,333 tokens / 128, +1 remainder)
n = 3 * C * m_chunk
raw = full[:n]
wl = bench.Workload("config3", n, 2025, C, 500_000_000, True, f"prefix of {C} chunks")
# extrapolation from bounded samples (the bench's own code path)
rs = bench.RefSampler(O, R, kind, raw, spum, wl, C, False)
for S in (8, 24, 8, 24):
    rs.sample(S)
ex = rs.extrapolate()
# the stock full-geometry run
cfg = O.make_cfg(workers=C, pub_path=spum)
t0 = time.perf_counter()
blob = R.compress(raw, cfg)
t1 = time.perf_counter()
out = R.decompress(blob, pub_path=spum, workers=C)
t2 = time.perf_counter()
assert out == raw
h = O.parse_container(blob)
print(json.dumps({"chunks": C, "bytes": n, "L": h["chunks"][0][1] // h["bs"],
                  "measured_compress_s": t1 - t0, "measured_decompress_s": t2 - t1,
                  "extrapolated_compress_s": ex["compress_s"], "extrapolated_decompress_s": ex["decompress_s"],
                  "ratio_extrapolated_over_measured": (ex["compress_s"] + ex["decompress_s"]) / (t2 - t0),
                  "per_step_ms": [ex["per_step_compress_s"] * 1e3, ex["per_step_decompress_s"] * 1e3],
                  "host_cores": os.cpu_count(), "kind": kind}))
