"""BASELINE config 4 at N=1 (one-off measurement, not the bench default):
10^9 B synthetic genome, default selector (> 500 MB => SPrM+DM, flags 6, with
the sequential SPrM pre-pass inside compress), SMP 0.05, W=256, defaults
otherwise. Device-resident input; compress and decompress timed with CUDA
events; lossless round trip checked."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2507_12805_b200 as P

n = int(float(sys.argv[1]) * 1e6) if len(sys.argv) > 1 else 10**9
W = int(sys.argv[2]) if len(sys.argv) > 2 else 256
t0 = time.time()
raw = P.synth("genome", n, 2026, 10)
cfg = P.CompressConfig(workers=W)
d_raw = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
tc, td = P.Timing(), P.Timing()
e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
torch.cuda.synchronize()
e[0].record()
blob = P.compress_device(d_raw.data_ptr(), n, cfg, tc)
e[1].record()
torch.cuda.synchronize()
e[2].record()
dptr, dlen = P.decompress_to_device(blob, "", 0, td)
e[3].record()
torch.cuda.synchronize()
out = P.decompress(blob, "")  # host API round trip check
ok = out == raw
P.device_free(dptr)
c_ms, d_ms = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3])
print(json.dumps({"config": "config4 (N=1)", "bytes": n, "W": W, "container_flags": blob[5],
                  "compress_MBps": n / 1e6 / (c_ms / 1e3), "decompress_MBps": n / 1e6 / (d_ms / 1e3),
                  "round_trip_MBps": n / 1e6 / ((c_ms + d_ms) / 1e3), "bits_per_base": 8 * len(blob) / n,
                  "sprm_prepass_ms": tc.sprm_ms, "compress_ticks_ms": tc.model_ms,
                  "decompress_ticks_ms": td.model_ms, "ticks": tc.ticks, "lossless": ok,
                  "wall_s": time.time() - t0}))
