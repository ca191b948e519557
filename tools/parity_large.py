"""Parity of the 1 GB workloads against the reference (SURVEY §8(c) parity
protocol step 5), run on the GPU box:

  config4  10^9 B synthetic genome (seed 2026), default selector (flags 6:
           SPrM pre-trained on the input inside compress), W=256
  config5  10^9 B species mixture (one GPU's share of the 10 GB config:
           160 source blocks, every 16th distribution-perturbed), W=256

1. The B200 compresses the input with stats, which export every chunk's
   inbound Step-wise Model Passing snapshot (WorkerStats::snapshot_recv_bytes),
   and decompresses it losslessly.
2. The reference itself (oracle/_ref) then checks, from those recorded
   snapshots and the container's own SPrM blob:
   * full chunks: encode_chunk_standalone (pipeline.cpp:298-301, the
     reference's own hook) of sampled chunks reproduces their payloads byte
     for byte;
   * SMP links: the reference's chunk replay of chunk c from its inbound
     snapshot, stopped at c's snapshot step, yields exactly the snapshot the
     B200 handed to chunk c+1 (its FNV-1a equals chunk c+1's recv hash).
The SPrM pre-pass itself (1.04 M sequential steps, ~38 h on one CPU core) is
pinned separately by tests/test_gpu_scale.py on its first 3,334 steps; here
both sides use the GPU-trained private model shipped in the container.

Usage: python tools/parity_large.py config4|config5 [full_chunks] [links]
Writes gpurun_out/parity_<config>.json."""
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracles as O  # noqa: E402
import paper_2507_12805_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "config4"
n_full = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n_links = int(sys.argv[3]) if len(sys.argv) > 3 else 16
n = 10**9
t0 = time.time()
if which == "config4":
    raw = P.synth("genome", n, 2026, 10)
else:
    raw = P.synth("species", n, 2026, max(1, int((64 << 20) * n / 1e10)))
cfg = P.CompressConfig(workers=256)
st = P.PipelineStats()
tc = time.time()
blob = P.compress(raw, cfg, st)
tc = time.time() - tc
td = time.time()
ok = P.decompress(blob) == raw
td = time.time() - td
h = O.parse_container(blob)
W = len(h["chunks"])
R = O.ref()
codes = np.frombuffer(raw, np.uint8)
codes = (((codes >> 1) ^ (codes >> 2)) & 3).astype(np.uint8).tobytes()
tok, _ = R.skmer_encode(codes, 3, 3)
del codes
bs, t = h["bs"], h["t"]


def chunk_tokens(c):
    ts, tl, _, _, _ = h["chunks"][c]
    L = tl // bs
    return np.ascontiguousarray(tok[ts:ts + bs * L]), L


def full(c):
    ct, _ = chunk_tokens(c)
    _, _, po, pl, _ = h["chunks"][c]
    pay = R.encode_chunk_standalone(ct, h["flags"], 3, t, bs, 4, h["dm_seed"], priv=h["priv"],
                                    inbound=st.workers[c].snapshot_recv_bytes)
    return {"chunk": c, "payload_len": pl, "identical": pay == blob[po:po + pl]}


def link(c):
    ct, L = chunk_tokens(c)
    snap = max(1, (h["myriad"] * L + 9999) // 10000)
    _, s = R.replay_chunk(ct, h["flags"], 3, t, bs, 4, h["dm_seed"], priv=h["priv"],
                          inbound=st.workers[c].snapshot_recv_bytes, snap_at=snap, stop_at=snap)
    want = st.workers[c + 1].snapshot_recv_hash
    return {"chunk": c, "snap_step": snap, "identical": O.fnv1a64(s) == want and want != 0}


picks_full = sorted({0, 1, W // 2, W - 1} | set(range(2, W, max(1, W // n_full))))[:n_full]
picks_link = [int(x) for x in np.linspace(0, W - 2, n_links).round()]
cores = os.cpu_count() or 1
tr = time.time()
with ThreadPoolExecutor(max_workers=cores) as ex:
    links = list(ex.map(link, picks_link))
    fulls = list(ex.map(full, picks_full))
tr = time.time() - tr
res = {"workload": which, "bytes": n, "chunks": W, "flags": h["flags"], "container_bytes": len(blob),
       "bits_per_base": 8.0 * len(blob) / n, "lossless_gpu_round_trip": ok,
       "gpu_compress_s_with_stats": tc, "gpu_decompress_s": td,
       "reference_full_chunk_recode": fulls, "reference_smp_links": links,
       "all_identical": all(x["identical"] for x in fulls + links),
       "reference_check_s": tr, "host_cores": cores, "wall_s": time.time() - t0}
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"parity_{which}.json").write_text(json.dumps(res, indent=1))
print(json.dumps({k: v for k, v in res.items() if k not in ("reference_full_chunk_recode",
                                                            "reference_smp_links")}))
